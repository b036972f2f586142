"""C-ABI boundary checks that need no GPU: the in-tree library loads, exports
every entry point include/poly_b200.h declares, and fails loudly (no CPU
fallback) when no CUDA device is present."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "poly_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(poly_b200_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1609_01882_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 15
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == declared


def test_cpp_header_compiles():
    import subprocess
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), "-x", "c++",
                        os.path.join(ROOT, "include", "poly_b200", "flat_index.hpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_no_cpu_fallback_without_gpu(pq8):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present; the GPU tests cover the device path")
    import paper_1609_01882_b200 as pb
    pq = pb.ProductQuantizer(8, 8, 128, pq8.codebooks, pq8.perms)
    with pytest.raises(pb.PolyError) as e:
        pb.FlatIndex(pq)
    assert e.value.code in (pb.Errc.invalid_argument, pb.Errc.internal)


def test_strategy_names():
    import paper_1609_01882_b200 as pb
    for s in ("adc", "binary", "disidx", "dual"):
        assert pb.to_string(pb.strategy_from_string(s)) == s
    with pytest.raises(pb.PolyError):
        pb.strategy_from_string("hamming")


def test_bench_and_entry_scripts_compile():
    """bench.py / __graft_entry__.py are driver contracts: they must at least compile."""
    import py_compile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for f in ("bench.py", "__graft_entry__.py"):
        py_compile.compile(os.path.join(root, f), doraise=True)
