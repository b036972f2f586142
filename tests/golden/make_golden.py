"""Generate the golden fixtures from the REFERENCE's own compiled sources.

Run here (where /root/reference exists):  python tests/golden/make_golden.py

Everything below is computed by ``oracle/_ref/libpolyref.so`` -- the reference
C++ sources compiled in place by ``oracle/Makefile`` -- except the synthetic
inputs, which come from the shared counter-based generator
(oracle/polyoracle.c ``po_gen_*``; GPU twin in csrc/synth.cuh).

Files:
  pq_d128_m8.npz   cfg 0/1 quantizer: 1000-center d=128 mixture, 100k train,
                   train_pq(m=8, dbits=8, 25 iters, seed 1234567) then
                   optimize_pq(defaults: distance loss, alpha 0.5, 500k iters)
  pq_d256_m16.npz  cfg 3 quantizer: 4096-center d=256 mixture, 100k train, m=16
  golden_m8.npz    known answers on pq_d128_m8: codes, LUTs, Hamming/ADC
                   matrices and search results for every strategy and tau
  golden_m16.npz   same for the 128-bit codes
  topk_kat.npz     the reference TopK's defect vs the SPEC contract
  golden_ivf.npz   IVF (no reference code): 64-cell coarse
                   quantizer from the reference's kmeans, residual PQ from
                   train_pq + optimize_pq on residuals, lists from the
                   reference's assign_nearest + encode, and search_coarse
                   results composed from reference primitives
                   (oracle/ref_driver.cpp ref_ivf_search)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
DATA_SEED = 160901882  # arXiv id; streams: 0 centers, 1 train, 2 base, 3 queries


def make_pq(name, dim, ncent, m, ntrain=100_000):
    path = os.path.join(OUT, name)
    if os.path.exists(path):
        z = np.load(path)
        return oracle.PQ(m, 8, dim, z["codebooks"], z["perms"])
    t = time.time()
    centers = oracle.gen_centers(DATA_SEED, ncent, dim)
    train = oracle.gen_points(DATA_SEED, 1, 0, ntrain, centers)
    cb = oracle.ref_train_pq(train, m, 8, 25, 1234567)
    perms = oracle.ref_optimize_pq(cb, dim)
    np.savez_compressed(path, codebooks=cb, perms=perms, dim=dim, m=m, dbits=8, ncent=ncent, ntrain=ntrain,
                        data_seed=DATA_SEED, recipe="ref train_pq(25 iters, seed 1234567) + optimize_pq defaults")
    print(f"{name}: trained in {time.time() - t:.1f}s")
    return oracle.PQ(m, 8, dim, cb, perms)


def make_golden(name, pq, ncent, n, nq, taus, normalize=False):
    centers = oracle.gen_centers(DATA_SEED, ncent, pq.dim)
    base = oracle.gen_points(DATA_SEED, 2, 0, n, centers, normalize)
    queries = oracle.gen_points(DATA_SEED, 3, 0, nq, centers, normalize)
    codes = oracle.ref_encode(pq, base)                 # pq.cpp:29-45
    codes_gemm = oracle.ref_encode_batch(pq, base)      # pq.cpp:47-78 (BLAS path)
    qcodes = oracle.ref_encode(pq, queries)
    lut, lutp = oracle.ref_compute_lut(pq, queries[:4])
    ham = oracle.ref_hamming_matrix(qcodes, codes[:2000]).astype(np.uint8)
    adc = oracle.ref_adc_matrix(pq, queries[:4], codes[:2000])
    out = dict(base_head=base[:64], queries=queries, codes=codes, codes_gemm=codes_gemm, qcodes=qcodes,
               lut=lut, lutp=lutp, ham=ham, adc=adc, data_seed=DATA_SEED, ncent=ncent, n=n)
    k = 100
    for strat in ("adc", "binary", "disidx"):
        i, s, c, _ = oracle.ref_search(pq, codes, queries, k, strategy=strat)
        out[f"{strat}_ids"], out[f"{strat}_scores"], out[f"{strat}_counts"] = i, s, c
    for tau in taus:
        i, s, c, sv = oracle.ref_search(pq, codes, queries, k, tau=tau, strategy="dual")
        out[f"dual{tau}_ids"], out[f"dual{tau}_scores"], out[f"dual{tau}_counts"], out[f"dual{tau}_surv"] = i, s, c, sv
    # small k and shortage / tie-heavy cases: 500 codes repeated 4x under shuffled ids
    rng = np.random.default_rng(7)
    tie_codes = np.repeat(codes[:500], 4, axis=0)
    tie_ids = rng.permutation(2000).astype(np.int64) * 3 + 11
    for tau in (taus[1], pq.code_bits):
        i, s, c, sv = oracle.ref_search(pq, tie_codes, queries, 7, tau=tau, ids=tie_ids)
        out[f"tie{tau}_ids"], out[f"tie{tau}_scores"], out[f"tie{tau}_counts"], out[f"tie{tau}_surv"] = i, s, c, sv
    out["tie_ids_in"] = tie_ids
    np.savez_compressed(os.path.join(OUT, name), **out)
    print(f"{name}: {n} codes, {nq} queries; encode vs encode_batch mismatches: "
          f"{int((codes != codes_gemm).any(axis=1).sum())}")


def make_topk_kat():
    # k=2 with offers 5,3,4,1 -> contract {1,3}; reference TopK returns {1,5}
    s = np.array([5, 3, 4, 1], np.float32)
    ids = np.arange(4, dtype=np.int64)
    bi, bs = oracle.ref_buggy_topk(s, ids, 2)
    rng = np.random.default_rng(1)
    trials = []
    for _ in range(200):
        n = int(rng.integers(1, 60))
        sc = rng.integers(0, 20, n).astype(np.float32)
        ii = rng.permutation(n).astype(np.int64)
        k = int(rng.integers(0, 12))
        want = sorted(zip(sc.tolist(), ii.tolist()))[:k]
        gi, gs = oracle.ref_buggy_topk(sc, ii, k)
        trials.append(list(zip(gs.tolist(), gi.tolist())) != want)
    np.savez_compressed(os.path.join(OUT, "topk_kat.npz"), offers=s, buggy_ids=bi, buggy_scores=bs,
                        buggy_mismatch_rate=np.float64(np.mean(trials)))
    print(f"topk_kat: reference TopK k=2 on 5,3,4,1 -> {bs.tolist()}; mismatch rate {np.mean(trials):.2f}")


def make_ivf_golden(name="golden_ivf.npz", nlist=64, ntrain=20000, n=20000, nq=24):
    t = time.time()
    centers = oracle.gen_centers(DATA_SEED, 1000, 128)
    train = oracle.gen_points(DATA_SEED, 1, 0, ntrain, centers)
    coarse = oracle.ref_kmeans(train, nlist, 10, 1234567)
    tr_assign = oracle.ref_assign_nearest(train, coarse)
    resid = train - coarse[tr_assign]
    cb = oracle.ref_train_pq(resid, 8, 8, 25, 1234567)
    perms = oracle.ref_optimize_pq(cb, 128)
    pq = oracle.PQ(8, 8, 128, cb, perms)
    base = oracle.gen_points(DATA_SEED, 2, 0, n, centers)
    assign_ref = oracle.ref_assign_nearest(base, coarse)          # distances.cpp:56-79 (GEMM)
    assign_exact = oracle.ivf_assign(base, coarse)                # sq_l2 argmin
    codes = oracle.ref_encode(pq, base - coarse[assign_ref])      # pq.cpp:29-45 on residuals
    order = np.argsort(assign_ref, kind="stable")
    off = np.zeros(nlist + 1, np.uint64)
    off[1:] = np.cumsum(np.bincount(assign_ref, minlength=nlist))
    lists = oracle.IVFLists(off, codes[order], order.astype(np.int64) * 7 + 3)
    queries = oracle.gen_points(DATA_SEED, 3, 0, nq, centers)
    out = dict(coarse=coarse, codebooks=cb, perms=perms, off=lists.off, list_codes=lists.codes, list_ids=lists.ids,
               assign_ref=assign_ref, assign_exact=assign_exact, queries=queries, base_head=base[:64],
               data_seed=DATA_SEED, n=n)
    for nprobe in (1, 4, 16, 64):
        for tau in (20, 26, 64):
            for cap in (0, 1500):
                i, sc, c, sv = oracle.ref_ivf_search(pq, coarse, lists, queries, 50, nprobe, tau=tau, cap=cap)
                key = f"p{nprobe}_t{tau}_c{cap}"
                out[key + "_ids"], out[key + "_scores"], out[key + "_counts"], out[key + "_surv"] = i, sc, c, sv
    for strat in ("adc", "binary"):
        i, sc, c, _ = oracle.ref_ivf_search(pq, coarse, lists, queries, 50, 16, strategy=strat)
        out[f"{strat}16_ids"], out[f"{strat}16_scores"], out[f"{strat}16_counts"] = i, sc, c
    np.savez_compressed(os.path.join(OUT, name), **out)
    print(f"{name}: nlist {nlist}, {n} codes in {time.time() - t:.1f}s; GEMM vs exact assignment mismatches: "
          f"{int((assign_ref != assign_exact).sum())}; list sizes {int(np.diff(off).min())}..{int(np.diff(off).max())}")


if __name__ == "__main__":
    oracle.build()
    pq8 = make_pq("pq_d128_m8.npz", 128, 1000, 8)
    pq16 = make_pq("pq_d256_m16.npz", 256, 4096, 16)
    make_golden("golden_m8.npz", pq8, 1000, 20000, 24, (0, 20, 24, 28, 32, 64))
    make_golden("golden_m16.npz", pq16, 4096, 10000, 16, (0, 48, 56, 64, 128))
    make_topk_kat()
    make_ivf_golden()
