// kernels_ivf.cu -- IVF search path (coarseindex; configs 2/4).
//
// The reference ships no IVF code; these kernels follow the oracle restatement
// (oracle/polyoracle.c po_ivf_*), itself pinned to golden vectors composed
// from the reference primitives:
//   K5  coarse_keys_kernel   sq_l2(q, c) (distances.cpp:10-17) for every cell, exact
//                            fp32 in dim order; key = (dist bits << 32 | cell), so K3
//                            with k = nprobe yields enumerate_cells:
//                            ascending distance, ties -> lower cell.
//   (the tensor-core form of enumerate_cells, K5t + K5q, is in kernels_coarse.cu)
//   K1r residual_lut_quad_kernel  per (query, probe): r = q - c_cell, then
//                            compute_lut / permuted_lut / encode on r
//                            (pq.cpp:29-45,91-119), packed f32x2, bit-exact.
//   K6  (kernels_ivf_scan.cu) the list scan over the probed cells.
//   assign_kernel            build: nearest coarse cell by sq_l2 (strict <).
#include <type_traits>

#include "code_ops.cuh"
#include "synth.cuh"

namespace pb {

// ------------------------------------------------------------------ K5
// CTA tile: 64 queries x 64 cells, 256 threads, 4 x 4 register block per thread;
// dims are consumed in chunks of 32 staged in shared memory.
constexpr int K5_T = 64, K5_D = 32;

__global__ void __launch_bounds__(256) coarse_keys_kernel(const float* __restrict__ q, uint32_t nq, uint32_t dim,
                                                          const float* __restrict__ cent, uint32_t nlist,
                                                          unsigned long long* __restrict__ keys) {
    __shared__ float qs[K5_T][K5_D + 1];
    __shared__ float cs[K5_T][K5_D + 1];
    const uint32_t c0 = blockIdx.x * K5_T, q0 = blockIdx.y * K5_T;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 each
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (uint32_t d0 = 0; d0 < dim; d0 += K5_D) {
        for (int e = threadIdx.x; e < K5_T * K5_D; e += 256) {
            const int r = e / K5_D, c = e % K5_D;
            qs[r][c] = (q0 + r < nq) ? q[(size_t)(q0 + r) * dim + d0 + c] : 0.0f;
            cs[r][c] = (c0 + r < nlist) ? cent[(size_t)(c0 + r) * dim + d0 + c] : 0.0f;
        }
        __syncthreads();
#pragma unroll 4
        for (int d = 0; d < K5_D; ++d) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = qs[ty + 16 * i][d];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = cs[tx + 16 * j][d];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float t = __fsub_rn(a[i], b[j]);
                    acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(t, t));  // sq_l2 order, no FMA
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t qi = q0 + ty + 16 * i;
        if (qi >= nq) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t c = c0 + tx + 16 * j;
            if (c < nlist) keys[(size_t)qi * nlist + c] = ((unsigned long long)__float_as_uint(acc[i][j]) << 32) | c;
        }
    }
}

void launch_coarse_keys(const float* q, uint32_t nq, uint32_t dim, const float* cent, uint32_t nlist,
                        unsigned long long* keys, cudaStream_t s) {
    if (nq == 0) return;
    dim3 grid((nlist + K5_T - 1) / K5_T, (nq + K5_T - 1) / K5_T);
    coarse_keys_kernel<<<grid, 256, 0, s>>>(q, nq, dim, cent, nlist, keys);
    count_launch();
}

// ------------------------------------------------------------------ K1r
// items (q, p) -> residual LUT (stored-field indexed) + code, all m sub-quantizers.
// One CTA per K1R_ITEMS consecutive items: thread j owns centroid j and loads its
// codebook row once per sub-quantizer for all the CTA's items (the 8 KB-per-sq
// codebook is the L2 traffic; the items share it).
#ifndef POLY_K1R_ITEMS
#define POLY_K1R_ITEMS 8
#endif
constexpr uint32_t K1R_ITEMS = POLY_K1R_ITEMS;
static_assert(K1R_ITEMS * 16 <= 128, "K1r writes the items' query codes with one thread per (item, sub-quantizer)");

// K1r, centroid pairs: thread t owns centroids t and t + 128 as one packed f32x2
// lane pair, so each (item, dim) term is FADD2 (r - c), FFMA2 (t * t + z, z a
// runtime +0.0: exactly mul.rn, and ptxas cannot contract it into the add), FADD2
// (acc + s) for two centroids -- the same rounding sequence as sq_l2 per lane.
// The residual sits in shared memory duplicated as (r, r) pairs.  (A pre-paired
// codebook layout that spares the register-pair MOVs measured slower: 381 -> 501 us.)
__device__ __forceinline__ unsigned long long k1_pack(float lo, float hi) {
    unsigned long long v;
    asm("mov.b64 %0, {%1,%2};" : "=l"(v) : "f"(lo), "f"(hi));
    return v;
}
// A packed pair that stays packed: the result of an FADD2 with a runtime -0.0 pair (x + -0.0 == x for
// every x).  ptxas rematerialises a plain mov.b64 pack at every use -- two MOVs per packed operand,
// 0.6 MOV per FP op in the term loop -- but keeps an arithmetic result in its register pair.
__device__ __forceinline__ unsigned long long k1_pack_once(float lo, float hi, unsigned long long nzz) {
    unsigned long long v;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(v) : "l"(k1_pack(lo, hi)), "l"(nzz));
    return v;
}

// K1r, two centroid pairs per thread: the 128 threads cover two sub-quantizers at a
// time (thread t: sq 2s + (t >> 6), pairs (u, u + 128) and (u + 64, u + 192), u = t & 63),
// so each shared-memory load of a residual pair feeds 12 packed FP ops instead of 6
// (the pair kernel's shared-memory pipe was 93% busy).
#ifndef POLY_K1R_MINB
#define POLY_K1R_MINB 5  // 94 registers, 5 CTAs per SM (A/B on config 4: 4 -> 686, 5 -> 659, 6 -> 702 us)
#endif
__global__ void __launch_bounds__(128, POLY_K1R_MINB) residual_lut_quad_kernel(const float* __restrict__ queries, uint32_t dim,
                                                                   uint32_t m,
                                                                   const unsigned long long* __restrict__ probe_keys,
                                                                   uint32_t nprobe, const uint32_t* __restrict__ items,
                                                                   const uint32_t* __restrict__ nitems_p,
                                                                   const float* __restrict__ cent,
                                                                   const float* __restrict__ codebooks,
                                                                   const uint16_t* __restrict__ perms,
                                                                   float* __restrict__ lutp,
                                                                   uint8_t* __restrict__ qcodes, float zero) {
    const uint32_t item0 = blockIdx.x * K1R_ITEMS, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t h = t >> 6, u = t & 63, wh = warp & 1;  // sub-quantizer half, pair index, warp within half
    const uint32_t nitems = *nitems_p;
    if (item0 >= nitems) return;
    const uint32_t ni = min(K1R_ITEMS, nitems - item0);
    auto gitem = [&](uint32_t i) { return __ldg(items + i); };  // global item q * nprobe + p
    __shared__ __align__(16) unsigned long long rr[K1R_ITEMS][256];  // (r, r) per dim
    __shared__ float wv[K1R_ITEMS][16][2];
    __shared__ uint32_t wj[K1R_ITEMS][16][2];
    __shared__ __align__(16) float stage[K1R_ITEMS][2][KSUB];  // two sub-quantizers' rows, stored-field order
    for (uint32_t e = t; e < ni * dim; e += 128) {
        const uint32_t it = e / dim, d = e % dim, item = gitem(item0 + it);
        const uint32_t qi = item / nprobe, cell = (uint32_t)probe_keys[item];
        const float r = __fsub_rn(queries[(size_t)qi * dim + d], cent[(size_t)cell * dim + d]);  // r = q - c
        rr[it][d] = k1_pack(r, r);
    }
    __syncthreads();
    const unsigned long long zz = k1_pack(zero, zero), nzz = k1_pack(-zero, -zero);
    const uint32_t ja = u, jb = u + 128, jc = u + 64, jd = u + 192;  // pair 0 = (ja, jb), pair 1 = (jc, jd)
    for (uint32_t s2 = 0; s2 < m / 2; ++s2) {
        const uint32_t sq = 2 * s2 + h;
        const float4* ca = reinterpret_cast<const float4*>(codebooks + ((size_t)sq * KSUB + ja) * DSUB);
        const float4* cb = reinterpret_cast<const float4*>(codebooks + ((size_t)sq * KSUB + jb) * DSUB);
        const float4* cc_ = reinterpret_cast<const float4*>(codebooks + ((size_t)sq * KSUB + jc) * DSUB);
        const float4* cd = reinterpret_cast<const float4*>(codebooks + ((size_t)sq * KSUB + jd) * DSUB);
        unsigned long long p0[DSUB], p1[DSUB];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const float4 a = __ldg(ca + v), b = __ldg(cb + v), c = __ldg(cc_ + v), d = __ldg(cd + v);
            p0[4 * v + 0] = k1_pack_once(a.x, b.x, nzz); p1[4 * v + 0] = k1_pack_once(c.x, d.x, nzz);
            p0[4 * v + 1] = k1_pack_once(a.y, b.y, nzz); p1[4 * v + 1] = k1_pack_once(c.y, d.y, nzz);
            p0[4 * v + 2] = k1_pack_once(a.z, b.z, nzz); p1[4 * v + 2] = k1_pack_once(c.z, d.z, nzz);
            p0[4 * v + 3] = k1_pack_once(a.w, b.w, nzz); p1[4 * v + 3] = k1_pack_once(c.w, d.w, nzz);
        }
        unsigned long long acc0[K1R_ITEMS], acc1[K1R_ITEMS];
#pragma unroll
        for (uint32_t it = 0; it < K1R_ITEMS; ++it) { acc0[it] = zz; acc1[it] = zz; }
#pragma unroll
        for (int d2 = 0; d2 < DSUB / 2; ++d2) {
#pragma unroll
            for (uint32_t it = 0; it < K1R_ITEMS; ++it) {
                const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(&rr[min(it, ni - 1)][sq * DSUB + 2 * d2]);
                unsigned long long tt, q2;
#define K1Q_TERM(XV, CV, ACC)                                                         \
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(tt) : "l"(XV), "l"(CV));                    \
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(q2) : "l"(tt), "l"(zz));               \
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(ACC) : "l"(ACC), "l"(q2));
                K1Q_TERM(x.x, p0[2 * d2], acc0[it])
                K1Q_TERM(x.x, p1[2 * d2], acc1[it])
                K1Q_TERM(x.y, p0[2 * d2 + 1], acc0[it])
                K1Q_TERM(x.y, p1[2 * d2 + 1], acc1[it])
#undef K1Q_TERM
            }
        }
        const uint32_t da = perms[sq * KSUB + ja], db = perms[sq * KSUB + jb];
        const uint32_t dc = perms[sq * KSUB + jc], dd = perms[sq * KSUB + jd];
        __syncthreads();  // the previous rows are written out
#pragma unroll
        for (uint32_t it = 0; it < K1R_ITEMS; ++it) {
            if (it >= ni) break;
            float va, vb, vc, vd;
            asm("mov.b64 {%0,%1}, %2;" : "=f"(va), "=f"(vb) : "l"(acc0[it]));
            asm("mov.b64 {%0,%1}, %2;" : "=f"(vc), "=f"(vd) : "l"(acc1[it]));
            stage[it][h][da] = va;
            stage[it][h][db] = vb;
            stage[it][h][dc] = vc;
            stage[it][h][dd] = vd;
            // argmin, ties -> lowest centroid (pq.cpp:38); index order ja < jc < jb < jd
            const uint32_t ba = __float_as_uint(va), bb = __float_as_uint(vb);
            const uint32_t bc = __float_as_uint(vc), bd = __float_as_uint(vd);
            const uint32_t wmin = __reduce_min_sync(0xffffffffu, min(min(ba, bb), min(bc, bd)));
            const uint32_t jj = ba == wmin ? ja : (bc == wmin ? jc : (bb == wmin ? jb : (bd == wmin ? jd : 0xFFFFFFFFu)));
            const uint32_t jmin = __reduce_min_sync(0xffffffffu, jj);
            if (lane == 0) { wv[it][sq][wh] = __uint_as_float(wmin); wj[it][sq][wh] = jmin; }
        }
        __syncthreads();
        for (uint32_t e = t; e < ni * 2 * (KSUB / 4); e += 128) {  // float4 rows out
            const uint32_t it = e / (2 * (KSUB / 4)), hh = (e / (KSUB / 4)) & 1, o = e % (KSUB / 4);
            reinterpret_cast<float4*>(lutp + ((size_t)gitem(item0 + it) * m + 2 * s2 + hh) * KSUB)[o] =
                reinterpret_cast<const float4*>(stage[it][hh])[o];
        }
    }
    __syncthreads();
    if (t < ni * m) {  // across the 2 warps of each sub-quantizer
        const uint32_t it = t / m, sq = t % m;
        float bv = wv[it][sq][0];
        uint32_t bj = wj[it][sq][0];
        if (wv[it][sq][1] < bv || (wv[it][sq][1] == bv && wj[it][sq][1] < bj)) bj = wj[it][sq][1];
        qcodes[(size_t)gitem(item0 + it) * m + sq] = static_cast<uint8_t>(perms[sq * KSUB + bj]);
    }
}

void launch_residual_lut(const float* queries, uint32_t dim, uint32_t m, const unsigned long long* probe_keys,
                         uint32_t nprobe, const uint32_t* items, const uint32_t* nitems, uint32_t max_items,
                         const float* cent, const float* codebooks, const uint16_t* perms, float* lutp,
                         uint8_t* qcodes, cudaStream_t s) {
    if (max_items == 0) return;
    const uint32_t grid = (max_items + K1R_ITEMS - 1) / K1R_ITEMS;  // CTAs past the device count exit
    residual_lut_quad_kernel<<<grid, 128, 0, s>>>(queries, dim, m, probe_keys, nprobe, items, nitems, cent, codebooks,
                                                  perms, lutp, qcodes, 0.0f);
    count_launch();
}

// ------------------------------------------------------------------ probes under the cap
// np_eff[q] = number of probes visited: stop after the probe at which the
// scanned count reaches cap (0 = no cap); scanned[q] = codes visited.
__global__ void ivf_probe_count_kernel(const unsigned long long* __restrict__ probe_keys, uint32_t nq,
                                       uint32_t nprobe, const uint64_t* __restrict__ off, uint64_t cap,
                                       uint32_t* __restrict__ np_eff, unsigned long long* __restrict__ scanned,
                                       uint32_t* __restrict__ split, uint64_t r1_codes, uint32_t r1_max,
                                       IvfWork w) {
    // one warp per query: list sizes in parallel, running prefix over the probes in order;
    // probe p is visited iff no cap or the codes before it are < cap
    const uint32_t qi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (qi >= nq) return;
    uint64_t base = 0;
    uint32_t ne = nprobe;
    for (uint32_t p0 = 0; p0 < nprobe; p0 += 32) {
        const uint32_t p = p0 + lane;
        uint64_t sz = 0;
        if (p < nprobe) {
            const uint32_t cell = (uint32_t)probe_keys[(size_t)qi * nprobe + p];
            sz = off[cell + 1] - off[cell];
        }
        uint64_t incl = sz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += v;
        }
        const uint64_t before = base + incl - sz;  // codes of probes < p
        const uint32_t stop = __ballot_sync(0xffffffffu, p < nprobe && cap && before >= cap);
        if (stop) {
            const uint32_t l = __ffs(stop) - 1;
            ne = p0 + l;
            base = __shfl_sync(0xffffffffu, before, l);
            break;
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
        np_eff[qi] = ne;
        scanned[qi] = base;
    }
    // round-1 split: the leading probes through the first one at which the round holds
    // >= r1_codes codes or r1_max non-empty lists (empty lists -- all the cells another rank
    // owns under by-list sharding -- do not count)
    if (split) {
        uint32_t sp = ne;
        uint64_t cum = 0;
        uint32_t nonempty = 0;
        for (uint32_t p0 = 0; p0 < ne; p0 += 32) {
            const uint32_t p = p0 + lane;
            uint64_t sz = 0;
            if (p < ne) {
                const uint32_t cell = (uint32_t)probe_keys[(size_t)qi * nprobe + p];
                sz = off[cell + 1] - off[cell];
            }
            uint64_t incl = sz;
            uint32_t incl_ne = sz > 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
                const uint32_t w = __shfl_up_sync(0xffffffffu, incl_ne, o);
                if (lane >= (uint32_t)o) {
                    incl += v;
                    incl_ne += w;
                }
            }
            const uint32_t hit = __ballot_sync(0xffffffffu, p < ne && (cum + incl >= r1_codes || nonempty + incl_ne >= r1_max));
            if (hit) {
                sp = p0 + __ffs(hit);
                break;
            }
            cum += __shfl_sync(0xffffffffu, incl, 31);
            nonempty += __shfl_sync(0xffffffffu, incl_ne, 31);
        }
        if (lane == 0) split[qi] = sp;
        // work lists: round 1 = probes [0, sp), round 2 = [sp, ne) (A/B: cutting round 1
        // at 2048 / 4096 rows instead of whole probes gained nothing).  Lists are cut into
        // chunks of w.chunk[r] rows; one item (query, probe, first list position, rows) per chunk.
        if (w.items[0]) {
            for (int r = 0; r < 2; ++r) {
                const uint32_t phi = r ? ne : sp, ch = w.chunk[r];
                for (uint32_t p0 = 0; p0 < phi; p0 += 32) {
                    const uint32_t p = p0 + lane;
                    uint32_t len = 0, pos = 0;  // the list's length and first position (< 2^32 codes per GPU)
                    if (p < phi) {
                        const uint32_t cell = (uint32_t)probe_keys[(size_t)qi * nprobe + p];
                        const uint64_t o0 = off[cell];
                        len = (uint32_t)(off[cell + 1] - o0);
                        pos = (uint32_t)o0;
                    }
                    // the round's non-empty items get a residual LUT (K1r)
                    const bool lut = p < phi && len > 0 && (r == 0 || p >= sp);
                    const uint32_t bl = __ballot_sync(0xffffffffu, lut);
                    if (bl) {
                        uint32_t base = 0;
                        if (lane == 0) base = atomicAdd(w.nlut + r, (uint32_t)__popc(bl));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (lut) w.lut_items[r][base + __popc(bl & ((1u << lane) - 1u))] = qi * nprobe + p;
                    }
                    const uint32_t ap = p < sp ? len : 0;  // round-1 rows of probe p
                    const uint32_t lo = r ? ap : 0, hi = r ? len : ap;
                    const uint32_t nch = hi > lo ? (hi - lo + ch - 1) / ch : 0;
                    uint32_t incl = nch;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= (uint32_t)o) incl += v;
                    }
                    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
                    uint32_t at = 0;
                    if (lane == 0 && tot) at = atomicAdd(w.nitems + r, tot);
                    at = __shfl_sync(0xffffffffu, at, 0) + incl - nch;
                    for (uint32_t c = 0; c < nch; ++c)
                        if (at + c < w.cap[r])
                            w.items[r][at + c] = make_uint4(qi, p, pos + lo + c * ch, min(hi, lo + (c + 1) * ch) - (lo + c * ch));
                        else
                            atomicOr(w.overflow, 1u);
                }
            }
        }
    }
}

void launch_ivf_probe_count(const unsigned long long* probe_keys, uint32_t nq, uint32_t nprobe, const uint64_t* off,
                            uint64_t cap, uint32_t* np_eff, unsigned long long* scanned, cudaStream_t s,
                            uint32_t* split, uint64_t r1_codes, uint32_t r1_max, const IvfWork& w) {
    if (nq == 0) return;
    ivf_probe_count_kernel<<<(nq * 32 + 127) / 128, 128, 0, s>>>(probe_keys, nq, nprobe, off, cap, np_eff, scanned,
                                                                  split, r1_codes, r1_max, w);
    count_launch();
}

// K6 (the list scan) is in kernels_ivf_scan.cu.

// ------------------------------------------------------------------ K6s
// Round-1 seed: a bound for round 1 itself, so that round 1 (which otherwise starts
// unbounded) appends few candidates.  One CTA per query scores the first `rows` codes of
// the query's first probed list exactly as K6 does (the item's LUT and query code from
// K1r) and sets thr[q] = min(thr[q], k-th key + 1) when it found >= k keys: the k-th key
// of a subset of round 1's codes is >= the k-th key of round 1 and of the final result,
// so the bound is valid; seed_compact still sets round 2's bound from round 1's exact k-th.
constexpr uint32_t K6S_THREADS = 256;

template <int M, int STRAT>
__global__ void __launch_bounds__(K6S_THREADS) ivf_seed_kernel(const IvfScanArgs a, uint32_t rows, uint32_t k) {
    using C = typename CodeT<M>::T;
    extern __shared__ __align__(16) uint8_t k6s_smem[];
    float* L = reinterpret_cast<float*>(k6s_smem);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(k6s_smem + M * KSUB * 4);
    __shared__ uint32_t cnt, hist[256], want_s;
    __shared__ unsigned long long prefix_s;
    const uint32_t q = blockIdx.x;
    const size_t item = (size_t)q * a.nprobe;  // the first probe
    const uint32_t cell = (uint32_t)a.probe_keys[item];
    const uint64_t beg = a.off[cell];
    const uint32_t n = (uint32_t)min((uint64_t)rows, a.off[cell + 1] - beg);
    if (n < k) return;  // fewer codes than k: no bound from this sample
    if (STRAT == DUAL || STRAT == ADC)
        for (uint32_t i = threadIdx.x; i < (uint32_t)M * KSUB / 4; i += K6S_THREADS)
            reinterpret_cast<float4*>(L)[i] = __ldg(reinterpret_cast<const float4*>(a.lutp + item * M * KSUB) + i);
    const C qc = reinterpret_cast<const C*>(a.qcodes)[item];
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const C* ci = reinterpret_cast<const C*>(a.codes) + beg;
    for (uint32_t i = threadIdx.x; i < n; i += K6S_THREADS) {
        const C code = ci[i];
        float score;
        if (strategy_score<M, STRAT>(L, code, qc, a.tau, 0xFFFFFFFFu, score))
            keys[atomicAdd(&cnt, 1u)] = ((unsigned long long)__float_as_uint(score) << 32) | __ldg(a.low + beg + i);
    }
    __syncthreads();
    const uint32_t nk = cnt;
    if (nk < k) return;
    unsigned long long prefix = 0, mask = 0;
    uint32_t want = k;
    for (int shift = 56; shift >= 0; shift -= 8) {
        hist[threadIdx.x] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < nk; i += K6S_THREADS) {
            const unsigned long long v = keys[i];
            if ((v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 0xFFu], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const uint32_t lane = threadIdx.x;
            uint32_t c[8], t = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c[j] = hist[lane * 8 + j];
                t += c[j];
            }
            uint32_t incl = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (uint32_t)o) incl += x;
            }
            const uint32_t excl = incl - t;
            if (excl < want && want <= incl) {
                uint32_t r = want - excl;
                int digit = lane * 8 + 7;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (r <= c[j]) {
                        digit = lane * 8 + j;
                        break;
                    }
                    r -= c[j];
                }
                prefix_s = prefix | ((unsigned long long)digit << shift);
                want_s = r;
            }
        }
        __syncthreads();
        prefix = prefix_s;
        want = want_s;
        mask |= 0xFFull << shift;
    }
    if (threadIdx.x == 0 && prefix + 1 < a.thr[q]) a.thr[q] = prefix + 1;  // prefix = the k-th key
}

template <int M, int STRAT>
static void launch_ivf_seed_m(const IvfScanArgs& a, uint32_t rows, uint32_t k, cudaStream_t s) {
    const size_t smem = (size_t)M * KSUB * 4 + (size_t)rows * 8;
    auto kfn = ivf_seed_kernel<M, STRAT>;
    set_max_smem((const void*)kfn, smem);
    kfn<<<a.nq, K6S_THREADS, smem, s>>>(a, rows, k);
    count_launch();
}

void launch_ivf_seed(const IvfScanArgs& a, int strategy, uint32_t m, uint32_t rows, uint32_t k, cudaStream_t s) {
    if (a.nq == 0 || rows == 0 || k == 0) return;
    const bool w = m == 16;
    switch (strategy) {
        case DUAL: w ? launch_ivf_seed_m<16, DUAL>(a, rows, k, s) : launch_ivf_seed_m<8, DUAL>(a, rows, k, s); break;
        case ADC: w ? launch_ivf_seed_m<16, ADC>(a, rows, k, s) : launch_ivf_seed_m<8, ADC>(a, rows, k, s); break;
        case BINARY: w ? launch_ivf_seed_m<16, BINARY>(a, rows, k, s) : launch_ivf_seed_m<8, BINARY>(a, rows, k, s); break;
        default: w ? launch_ivf_seed_m<16, DISIDX>(a, rows, k, s) : launch_ivf_seed_m<8, DISIDX>(a, rows, k, s); break;
    }
}

// ------------------------------------------------------------------ build
// Nearest coarse cell of each vector (sq_l2, strict <, ties -> lowest cell);
// cells are staged through shared memory 32 at a time.
__global__ void __launch_bounds__(128) assign_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim,
                                                     const float* __restrict__ cent, uint32_t nlist,
                                                     uint32_t* __restrict__ assign) {
    extern __shared__ float cs[];  // 32 x dim
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < n;
    float best = 0.0f;
    uint32_t bi = 0;
    for (uint32_t c0 = 0; c0 < nlist; c0 += 32) {
        const uint32_t nc = min(32u, nlist - c0);
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < nc * dim; e += blockDim.x) cs[e] = cent[(size_t)c0 * dim + e];
        __syncthreads();
        if (!live) continue;
        for (uint32_t c = 0; c < nc; ++c) {
            float acc = 0.0f;
            for (uint32_t d = 0; d < dim; ++d) {
                const float t = __fsub_rn(x[i * dim + d], cs[c * dim + d]);
                acc = __fadd_rn(acc, __fmul_rn(t, t));
            }
            if ((c0 == 0 && c == 0) || acc < best) { best = acc; bi = c0 + c; }
        }
    }
    if (live) assign[i] = bi;
}

void launch_assign(const float* x, uint64_t n, uint32_t dim, const float* cent, uint32_t nlist, uint32_t* assign,
                   cudaStream_t s) {
    if (n == 0) return;
    assign_kernel<<<(unsigned)((n + 127) / 128), 128, 32 * dim * sizeof(float), s>>>(x, n, dim, cent, nlist, assign);
    count_launch();
}

// Residual codes encode(x - c_assign) (pq.cpp:29-45 on residuals), one thread per vector.
__global__ void __launch_bounds__(128) residual_encode_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim,
                                                              uint32_t m, const float* __restrict__ cent,
                                                              const uint32_t* __restrict__ assign,
                                                              const float* __restrict__ codebooks,
                                                              const uint16_t* __restrict__ perms,
                                                              uint8_t* __restrict__ codes) {
    __shared__ float4 cb[KSUB * DSUB / 4];
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < n;
    const float* cr = live ? cent + (size_t)assign[i] * dim : cent;
    for (uint32_t sq = 0; sq < m; ++sq) {
        __syncthreads();
        const float4* src = reinterpret_cast<const float4*>(codebooks + (size_t)sq * KSUB * DSUB);
        for (int e = threadIdx.x; e < KSUB * DSUB / 4; e += blockDim.x) cb[e] = src[e];
        __syncthreads();
        if (!live) continue;
        float r[DSUB];
#pragma unroll
        for (int t = 0; t < DSUB; ++t) r[t] = __fsub_rn(x[i * dim + sq * DSUB + t], cr[sq * DSUB + t]);
        uint32_t best = 0;
        float best_d = 0.0f;
        for (uint32_t j = 0; j < KSUB; ++j) {
            float acc = 0.0f;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const float4 cc = cb[j * 4 + v];
                float t;
                t = __fsub_rn(r[4 * v + 0], cc.x); acc = __fadd_rn(acc, __fmul_rn(t, t));
                t = __fsub_rn(r[4 * v + 1], cc.y); acc = __fadd_rn(acc, __fmul_rn(t, t));
                t = __fsub_rn(r[4 * v + 2], cc.z); acc = __fadd_rn(acc, __fmul_rn(t, t));
                t = __fsub_rn(r[4 * v + 3], cc.w); acc = __fadd_rn(acc, __fmul_rn(t, t));
            }
            if (j == 0 || acc < best_d) { best_d = acc; best = j; }
        }
        codes[i * m + sq] = static_cast<uint8_t>(perms[sq * KSUB + best]);
    }
}

void launch_residual_encode(const float* x, uint64_t n, uint32_t dim, uint32_t m, const float* cent,
                            const uint32_t* assign, const float* codebooks, const uint16_t* perms, uint8_t* codes,
                            cudaStream_t s) {
    if (n == 0) return;
    residual_encode_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(x, n, dim, m, cent, assign, codebooks, perms,
                                                                        codes);
    count_launch();
}

// Synthetic rows [row0, row0 + n) of the mixture, written as floats (chunked build).
// (launch_gen_points in kernels_encode.cu does this.)

// CSR bucketing: histogram of cells, then scatter (order within a list is
// irrelevant: results order by (score, id), never by list position).
__global__ void cell_hist_kernel(const uint32_t* __restrict__ assign, uint64_t n, unsigned long long* __restrict__ hist) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&hist[assign[i]], 1ull);
}

__global__ void cell_scatter_kernel(const uint32_t* __restrict__ assign, uint64_t n, uint32_t cb,
                                    const uint8_t* __restrict__ codes_in, const uint32_t* __restrict__ low_in,
                                    unsigned long long* __restrict__ cursor, uint8_t* __restrict__ codes_out,
                                    uint32_t* __restrict__ low_out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t at = atomicAdd(&cursor[assign[i]], 1ull);
        for (uint32_t b = 0; b < cb; b += 8)
            *reinterpret_cast<uint2*>(codes_out + at * cb + b) = *reinterpret_cast<const uint2*>(codes_in + i * cb + b);
        low_out[at] = low_in[i];
    }
}

void launch_cell_hist(const uint32_t* assign, uint64_t n, unsigned long long* hist, cudaStream_t s) {
    if (n == 0) return;
    cell_hist_kernel<<<148 * 4, 256, 0, s>>>(assign, n, hist);
    count_launch();
}

void launch_cell_scatter(const uint32_t* assign, uint64_t n, uint32_t cb, const uint8_t* codes_in,
                         const uint32_t* low_in, unsigned long long* cursor, uint8_t* codes_out, uint32_t* low_out,
                         cudaStream_t s) {
    if (n == 0) return;
    cell_scatter_kernel<<<148 * 4, 256, 0, s>>>(assign, n, cb, codes_in, low_in, cursor, codes_out, low_out);
    count_launch();
}

// key low word of insertion position i: id0 + i (arithmetic ids) or id32[i].
__global__ void key_low_kernel(uint64_t n, int mode, uint32_t id0, const uint32_t* __restrict__ id32,
                               uint32_t* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = mode == ID_ARITH ? id0 + (uint32_t)i : id32[i];
}

void launch_key_low(uint64_t n, int mode, uint32_t id0, const uint32_t* id32, uint32_t* out, cudaStream_t s) {
    if (n == 0) return;
    key_low_kernel<<<148 * 4, 256, 0, s>>>(n, mode, id0, id32, out);
    count_launch();
}

}  // namespace pb
