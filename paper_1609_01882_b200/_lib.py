"""ctypes binding of libpoly_b200.so (include/poly_b200.h).

The library is built in-tree by ``paper_1609_01882_b200.build``.  There is no
fallback: if the shared library is missing or fails to load, importing the
package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("POLY_B200_LIB") or os.path.join(HERE, "libpoly_b200.so")  # env: experiments only

_P = C.c_void_p
_u32, _u64, _i32, _f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_double


class PqDesc(C.Structure):
    _fields_ = [("m", _u32), ("dbits", _u32), ("dim", _u64), ("codebooks", _P), ("perms", _P)]


class SearchParamsC(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("k", _u32), ("tau", _u32)]


class IvfParamsC(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("k", _u32), ("tau", _u32), ("nprobe", _u32), ("cap", _u64)]


class SearchStatsC(C.Structure):
    _fields_ = [("scanned", _u64), ("survivors", _u64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1609_01882_b200/build.py` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.poly_b200_last_error.restype = C.c_char_p
    L.poly_b200_create.argtypes = [C.POINTER(PqDesc), _i32, C.POINTER(_P)]
    L.poly_b200_destroy.argtypes = [_P]
    L.poly_b200_size.argtypes = [_P]
    L.poly_b200_size.restype = _u64
    L.poly_b200_code_bytes.argtypes = [_P]
    L.poly_b200_code_bytes.restype = _u32
    L.poly_b200_add.argtypes = [_P, _P, _u64, _P]
    L.poly_b200_add_codes.argtypes = [_P, _P, _P, _u64]
    L.poly_b200_search_batch.argtypes = [_P, _P, _u64, C.POINTER(SearchParamsC), _P, _P, _P,
                                         C.POINTER(SearchStatsC)]
    L.poly_b200_search_batch_device.argtypes = [_P, _P, _u64, C.POINTER(SearchParamsC), _P, _P, _P, _P, _P,
                                                C.POINTER(SearchStatsC)]
    L.poly_b200_search_batch_device_ex.argtypes = [_P, _P, _u64, C.POINTER(SearchParamsC), _P, _P, _P, _P, _P, _P,
                                                   C.POINTER(SearchStatsC)]
    L.poly_b200_calibrate_threshold.argtypes = [_P, _P, _u64, _f64, C.POINTER(_u32), C.POINTER(_i32)]
    L.poly_b200_with_assignments.argtypes = [_P, _P, C.POINTER(_P)]
    L.poly_b200_get_codes.argtypes = [_P, _P, _P]
    L.poly_b200_search_keys_device.argtypes = [_P, _P, _u64, C.POINTER(SearchParamsC), _P, _P, _P, _P]
    L.poly_b200_merge_keys_device.argtypes = [_P, _P, _P, _u32, _u64, _u32, _P, _P, _P, _P]
    L.poly_b200_add_synthetic.argtypes = [_P, _u64, _P, _u32, _u32, _u64, _u64, _i32]
    L.poly_b200_gen_points_device.argtypes = [_i32, _u64, _P, _u32, _u32, _u32, _u64, _u64, _i32, _P, _P]
    L.poly_b200_debug_lut.argtypes = [_P, _P, _u64, _P, _P]
    L.poly_b200_debug_counts.argtypes = [_P, _P, _P, _u32]
    L.poly_b200_debug_set_list_capacity.argtypes = [_P, _u32]
    L.poly_b200_debug_rescued.argtypes = [_P, C.POINTER(_u32)]
    L.poly_b200_ivf_debug_set_list_capacity.argtypes = [_P, _u32]
    L.poly_b200_sharded_create.argtypes = [C.POINTER(PqDesc), _P, _u32, C.POINTER(_P)]
    L.poly_b200_sharded_destroy.argtypes = [_P]
    L.poly_b200_sharded_size.argtypes = [_P]
    L.poly_b200_sharded_size.restype = _u64
    L.poly_b200_sharded_count.argtypes = [_P]
    L.poly_b200_sharded_count.restype = _u32
    L.poly_b200_sharded_shard_size.argtypes = [_P, _u32, C.POINTER(_u64)]
    L.poly_b200_sharded_add.argtypes = [_P, _P, _u64, _P]
    L.poly_b200_sharded_add_codes.argtypes = [_P, _P, _P, _u64]
    L.poly_b200_sharded_search_batch.argtypes = [_P, _P, _u64, C.POINTER(SearchParamsC), _P, _P, _P,
                                                 C.POINTER(SearchStatsC)]
    L.poly_b200_kmeans.argtypes = [_P, _u64, _u32, _u32, _u32, _u64, _i32, _P, _P, _P, C.POINTER(_f64)]
    L.poly_b200_knn_writer_open.argtypes = [C.c_char_p, C.c_char_p, _u32, C.POINTER(_P)]
    L.poly_b200_ivf_knn_graph_write_device.argtypes = [_P, _P, _P, _u64, C.c_int64, C.POINTER(IvfParamsC), _P]
    L.poly_b200_knn_writer_close.argtypes = [_P, C.POINTER(_u64)]
    L.poly_b200_ivf_set_batch.argtypes = [_P, _u32]
    L.poly_b200_ivf_batch.argtypes = [_P]
    L.poly_b200_ivf_batch.restype = _u32
    L.poly_b200_ivf_save.argtypes = [_P, C.c_char_p]
    L.poly_b200_ivf_load.argtypes = [C.c_char_p, _i32, C.POINTER(_P)]
    L.poly_b200_ivf_get_cells.argtypes = [_P, _P, _u32, _P, _P, _P]
    L.poly_b200_ivf_profile_enable.argtypes = [_P, _i32]
    L.poly_b200_ivf_profile_read.argtypes = [_P, C.POINTER(_f64), C.POINTER(_u64)]
    L.poly_b200_ivf_debug_rescued.argtypes = [_P, C.POINTER(_u32)]
    L.poly_b200_profile_enable.argtypes = [_P, _i32]
    L.poly_b200_profile_read.argtypes = [_P, C.POINTER(_f64), C.POINTER(_u64)]
    L.poly_b200_launch_count.restype = _u64
    L.poly_b200_ivf_create.argtypes = [C.POINTER(PqDesc), _P, _u32, _i32, C.POINTER(_P)]
    L.poly_b200_ivf_destroy.argtypes = [_P]
    L.poly_b200_ivf_size.argtypes = [_P]
    L.poly_b200_ivf_size.restype = _u64
    L.poly_b200_ivf_assign.argtypes = [_P, _P, _u64, _P]
    L.poly_b200_ivf_add.argtypes = [_P, _P, _u64, _P, _P]
    L.poly_b200_ivf_add_device.argtypes = [_P, _P, _P, _u64, C.c_int64, _P]
    L.poly_b200_ivf_add_device_ids.argtypes = [_P, _P, _P, _u64, _P, _P]
    L.poly_b200_ivf_search_keys_phase_device.argtypes = [_P, _P, _u64, C.POINTER(IvfParamsC), _P, _i32, _P, _P, _P,
                                                         _P, C.POINTER(SearchStatsC)]
    L.poly_b200_ivf_add_codes.argtypes = [_P, _P, _P, _P, _u64]
    L.poly_b200_ivf_get_lists.argtypes = [_P, _P, _P, _P]
    L.poly_b200_ivf_probes.argtypes = [_P, _P, _u64, _u32, _P]
    L.poly_b200_ivf_search.argtypes = [_P, _P, _u64, C.POINTER(IvfParamsC), _P, _P, _P, C.POINTER(SearchStatsC)]
    L.poly_b200_ivf_search_device.argtypes = [_P, _P, _u64, C.POINTER(IvfParamsC), _P, _P, _P, _P,
                                              C.POINTER(SearchStatsC)]
    L.poly_b200_ivf_search_device_ex.argtypes = [_P, _P, _u64, C.POINTER(IvfParamsC), _P, _P, _P, _P, _P, _P,
                                                 C.POINTER(SearchStatsC)]
    L.poly_b200_ivf_knn_graph_device.argtypes = [_P, _P, _u64, C.c_int64, C.POINTER(IvfParamsC), _P, _P, _P, _P]
    L.poly_b200_ivf_search_keys_device.argtypes = [_P, _P, _u64, C.POINTER(IvfParamsC), _P, _P, _P,
                                                   C.POINTER(SearchStatsC)]
    L.poly_b200_ivf_merge_keys_device.argtypes = [_P, _P, _P, _u32, _u64, _u32, _P, _P, _P, _P]
    L.poly_b200_ivf_probe_keys_device.argtypes = [_P, _P, _u64, _u32, _P, _P]
    L.poly_b200_ivf_search_keys_probes_device.argtypes = [_P, _P, _u64, C.POINTER(IvfParamsC), _P, _P, _P, _P,
                                                          C.POINTER(SearchStatsC)]
    return L


lib = _load()

# names the C ABI exports (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "poly_b200_last_error", "poly_b200_create", "poly_b200_destroy", "poly_b200_size", "poly_b200_code_bytes",
    "poly_b200_add", "poly_b200_add_codes", "poly_b200_search_batch", "poly_b200_search_batch_device",
    "poly_b200_search_batch_device_ex", "poly_b200_ivf_search_device_ex", "poly_b200_debug_set_list_capacity",
    "poly_b200_debug_rescued", "poly_b200_ivf_debug_set_list_capacity", "poly_b200_ivf_debug_rescued",
    "poly_b200_ivf_get_cells", "poly_b200_ivf_profile_enable", "poly_b200_ivf_profile_read", "poly_b200_ivf_save",
    "poly_b200_ivf_load", "poly_b200_ivf_set_batch", "poly_b200_ivf_batch",
    "poly_b200_sharded_create", "poly_b200_sharded_destroy", "poly_b200_sharded_size", "poly_b200_sharded_count",
    "poly_b200_sharded_shard_size", "poly_b200_sharded_add", "poly_b200_sharded_add_codes",
    "poly_b200_sharded_search_batch", "poly_b200_knn_writer_open", "poly_b200_ivf_knn_graph_write_device",
    "poly_b200_knn_writer_close", "poly_b200_kmeans", "poly_b200_ivf_add_device_ids",
    "poly_b200_ivf_search_keys_phase_device",
    "poly_b200_calibrate_threshold", "poly_b200_with_assignments", "poly_b200_get_codes",
    "poly_b200_search_keys_device", "poly_b200_merge_keys_device", "poly_b200_add_synthetic",
    "poly_b200_gen_points_device", "poly_b200_debug_lut", "poly_b200_debug_counts", "poly_b200_profile_enable", "poly_b200_profile_read",
    "poly_b200_launch_count", "poly_b200_ivf_create", "poly_b200_ivf_destroy", "poly_b200_ivf_size",
    "poly_b200_ivf_assign", "poly_b200_ivf_add", "poly_b200_ivf_add_device", "poly_b200_ivf_add_codes",
    "poly_b200_ivf_get_lists", "poly_b200_ivf_probes", "poly_b200_ivf_search", "poly_b200_ivf_search_device", "poly_b200_ivf_knn_graph_device",
    "poly_b200_ivf_search_keys_device", "poly_b200_ivf_merge_keys_device", "poly_b200_ivf_probe_keys_device",
    "poly_b200_ivf_search_keys_probes_device",
]
