"""B200-native polysemous-code search (arXiv 1609.01882), drop-in for the
reference's flat index (poly::FlatIndex, flat_index.hpp:99-144).

Host mirror in Python (this package) and C++ (include/poly_b200/flat_index.hpp)
over the C ABI of libpoly_b200.so (include/poly_b200.h); hand-written sm_100a
kernels in csrc/.  See DESIGN.md.
"""
from .flat_index import (Errc, FlatIndex, Neighbor, PolyError, ProductQuantizer, SearchParams, SearchStats,
                         ShardedFlatIndex, Strategy, gen_points_device, launch_count, strategy_from_string, to_string)

from .ivf_index import CoarseParams, IVFIndex, KnnGraphWriter, kmeans

__all__ = ["CoarseParams", "IVFIndex", "KnnGraphWriter", "kmeans", "Errc", "FlatIndex", "Neighbor", "PolyError", "ProductQuantizer", "SearchParams", "SearchStats",
           "ShardedFlatIndex", "Strategy", "gen_points_device", "launch_count", "strategy_from_string", "to_string"]
