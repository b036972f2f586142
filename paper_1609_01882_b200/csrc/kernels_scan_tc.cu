// kernels_scan_tc.cu -- K2t: the flat dual scan for 64-bit codes (m = 8) with the
// Hamming filter on the tensor cores and the work split by role (sm_100a).
//
// Same arithmetic as K2 (kernels_scan.cu; hamming_bytes flat_index.hpp:14-27 as an
// int8 tcgen05.mma whose sign is exactly [h <= tau]; adc_distance
// pq.cpp:121-128 with __fadd_rn in sub-quantizer order; candidate keys against the
// query bound, exact top-k in K3), different schedule.  In K2 every consumer warp
// both feeds the MMA and drains its own survivors, and a quad's MMA waits for the
// slowest of its four warps' survivor work: ~1/3 of the issued instructions were
// polls.  Here the roles are separate warps of one persistent CTA per SM:
//
//   producer (1 warp)   TMA ring of code tiles (cp.async.bulk + mbarriers), serves
//                       the threshold selects, refreshes the bounds (as K2);
//   filter (FQ quads)   per half-step (128 codes = 4 warps x 32 lanes, one code per
//                       lane): expand each code into 64 e2m1 elements (bit -> 0.5) in
//                       a shared-memory A tile, preload the accumulator with the
//                       per-query bias |q| - tau - 1/2, and one elected thread issues
//                       ONE block-scaled MMA (kind::mxf4, M = 128, N = 16, K = 64,
//                       unit ue8m0 scales): D = |x| - 2<x,q> + |q| - tau - 1/2 =
//                       h - tau - 1/2, so sign(D) = [h <= tau] exactly (small
//                       integers + 1/2 in fp32).  The warps read D back and write each
//                       warp's 64-code x 16-query survivor mask (one word per lane) to
//                       a mask slot in shared memory.  Two accumulators per quad keep
//                       two MMAs in flight; the work is uniform, so the quad's warps
//                       stay in step without waiting on survivors.  (The int8 form of
//                       K2 needs 3 MMAs per 128 codes; a tcgen05.mma costs ~70 clk of
//                       tensor pipe per instruction here whatever N <= 128 is,
//                       tools/umma_rate.cu, so K = 64 bits in one instruction is 3x
//                       less tensor time per code.)
//   drain (the rest)    claim mask slots in order, compact the survivor bits into a
//                       per-warp queue, ADC + candidate test 32 at a time, and
//                       release the tile stage once all its slots are drained.
//
// Slot k of a tile holds codes [64 k, 64 k + 64): bit q of lane l is code 64 k + l
// against query q, bit 16 + q code 64 k + l + 32 (K2's TC layout), so the drain code
// is K2's.  A slot is handed over by an mbarrier per (stage, slot); its parity is the
// tile stage's use count.
#include "scan_common.cuh"

namespace pb {

#ifndef POLY_K2T_FQ  // filter quads
#define POLY_K2T_FQ 3
#endif
#ifndef POLY_K2T_RING
#define POLY_K2T_RING 160
#endif
#ifndef POLY_K2T_DEBUG  // 1: no MMA (the accumulator keeps its bias preload; debug only)
#define POLY_K2T_DEBUG 0
#endif
#ifndef POLY_K2T_STG
#define POLY_K2T_STG 3
#endif

namespace k2t {
constexpr int M = 8, Q = 16;
constexpr int FQ = POLY_K2T_FQ;
constexpr int NBUF = 2;                // accumulators (and A tiles) per filter quad
constexpr int NW = 32;                 // warps per CTA
constexpr int NF = 4 * FQ;             // filter warps: 0 .. NF-1
constexpr int PROD = NW - 1;           // producer warp
constexpr int ND = NW - 1 - NF;        // drain warps: NF .. NW-2
constexpr int STG = POLY_K2T_STG;   // tile ring depth
constexpr int TC = TILE_BYTES / M;     // codes per tile
constexpr int NSLOT = TC / 64;         // mask slots per tile (one per 64 codes)
constexpr int HSTEPS = NSLOT / 2;      // half-steps (128 codes) per tile
constexpr int RING = POLY_K2T_RING;
constexpr int PART_BITS = RING >= 32 + 256 ? 8 : 4;
constexpr uint32_t A_BYTES = 128 * 32;  // one MMA's A tile: 128 codes x 64 e2m1
constexpr uint32_t B_BYTES = 16 * 32;   // 16 queries x 64 e2m1
constexpr uint32_t SF_COL = 0;          // TMEM columns [0, 32): unit scale factors (A at 0, B at 16)
constexpr uint32_t D_COL = 32;          // accumulators: quad f, buffer b at D_COL + 16 (2 f + b)
static_assert(NSLOT % 4 == 0, "a tile must split into whole quad-steps");
static_assert(RING >= 32 + 32 * PART_BITS, "ring must hold a remainder plus one mask part");
static_assert(D_COL + 16 * NBUF * FQ <= 128, "TMEM budget (128 columns allocated)");
static_assert(ND >= 1, "no drain warps");
constexpr int LS = M * KSUB + 1;       // floats per query LUT (+1: bank skew, as K2)
constexpr size_t LUT_BYTES = (size_t)Q * LS * 4;
constexpr size_t TILES = (size_t)STG * TILE_BYTES;
constexpr size_t MASKS = (size_t)STG * NSLOT * 32 * 4;
constexpr size_t RINGS = (size_t)ND * RING * 4;
constexpr size_t AOFF = (LUT_BYTES + TILES + MASKS + RINGS + 1023) & ~(size_t)1023;
constexpr size_t TOTAL = AOFF + (size_t)FQ * NBUF * A_BYTES + B_BYTES;
// kind::mxf4 instruction descriptor: A, B e2m1 (1), K-major, N = 16, ue8m0 scales, M = 128, K = 64
constexpr uint32_t IDESC_MXF4_M128_N16 = (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
}  // namespace k2t

template <bool PERQ>
__global__ void __launch_bounds__(k2t::NW * 32, 1) scan_tc_kernel(const ScanArgs a) {
    using namespace k2t;
    using C = uint2;
    constexpr int NT = NW * 32;
    const uint32_t bs = a.bs;
    extern __shared__ __align__(128) uint8_t smem[];
    float* lut = reinterpret_cast<float*>(smem);
    C* tiles = reinterpret_cast<C*>(smem + LUT_BYTES);
    uint32_t* masks = reinterpret_cast<uint32_t*>(smem + LUT_BYTES + TILES);
    uint32_t* rings = reinterpret_cast<uint32_t*>(smem + LUT_BYTES + TILES + MASKS);

    __shared__ __align__(8) uint64_t full_bar[STG];
    __shared__ __align__(8) uint64_t empty_bar[STG];
    __shared__ __align__(8) uint64_t slot_bar[STG * NSLOT];
    __shared__ __align__(8) uint64_t qbar_s[FQ * NBUF];
    __shared__ unsigned long long thr_s[Q];
    __shared__ uint32_t surv_s[Q];
    __shared__ unsigned long long hash_s[PERQ ? Q : 1];
    __shared__ uint32_t unit_s, nreq_s, group_s, dclaim_s, req_head_s, cg_s, tmem_s;
    __shared__ uint32_t req_s[MAXREQ];
    __shared__ uint32_t sel_hist[256];
    
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STG; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], NSLOT);
        }
        for (int i = 0; i < STG * NSLOT; ++i) mbar_init(&slot_bar[i], 2);  // two filter warps per slot
        for (int i = 0; i < FQ * NBUF; ++i) mbar_init(&qbar_s[i], 1);
        fence_mbar_init();
        nreq_s = 0;
        req_head_s = 0;
        group_s = 0xFFFFFFFFu;
        cg_s = blockIdx.x % a.ngroups;
    }
    if (threadIdx.x < MAXREQ) req_s[threadIdx.x] = 0xFFFFFFFFu;
    if (warp == 0) tmem_alloc(&tmem_s, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_s;
    const uint32_t tlane = (uint32_t)(32 * (warp & 3)) << 16;
    if (warp < 4) {  // unit scale factors (ue8m0 127 = 1.0) in every byte of the SF columns
        for (uint32_t c = 0; c < 32; c += 8) tmem_st8(tbase + tlane + SF_COL + c, 0x7F7F7F7Fu);
        tmem_wait_st();
    }
    tc_fence_before();
    uint8_t* const bq_s = smem + AOFF + (size_t)FQ * NBUF * A_BYTES;  // B: the group's query weights

    uint32_t seq = 0;            // tiles consumed before this unit (all roles)
    uint32_t fstep = 0;          // filter warps: half-steps done by this warp (all units)
    float bias[Q];               // filter warps: accumulator preload |q| - tau - 1/2 per query
    const uint32_t tile_base = smem_u32(tiles), mask_base = smem_u32(masks), lut_base = smem_u32(lut);

    auto serve_selects = [&]() {  // producer warp: threshold selects requested by the appends
        for (;;) {
            uint32_t req = 0xFFFFFFFFu;
            if (lane == 0) {
                const uint32_t tail = *(volatile uint32_t*)&nreq_s;
                if (tail - req_head_s > MAXREQ) req_head_s = tail - MAXREQ;  // dropped requests
                if (req_head_s != tail) {
                    volatile uint32_t* slot = &req_s[req_head_s % MAXREQ];
                    req = *slot;
                    if (req != 0xFFFFFFFFu) {
                        *slot = 0xFFFFFFFFu;
                        ++req_head_s;
                    }
                }
            }
            req = __shfl_sync(0xffffffffu, req, 0);
            if (req == 0xFFFFFFFFu) break;
            const uint32_t qg = req >> 16, blk = req & 0xFFFFu;
            if (qg >= a.nqb || blk >= a.cap / bs) continue;
            __threadfence();
            const unsigned long long kth =
                warp_select_kth(a.cand + (size_t)qg * a.cap + (size_t)blk * bs, bs, a.k, sel_hist);
            if (lane == 0) atomicMin(a.thr + qg, kth);
        }
    };

    for (;;) {
        if (threadIdx.x == 0) {  // next unit: K2's group-affine schedule with a bounded lead
            uint32_t g = cg_s, u = a.units;
            if (a.affine) {
                for (uint32_t tries = 0; tries < 4 * a.ngroups + 4; ++tries) {
                    uint32_t gmin = g, cmin = 0xFFFFFFFFu;
                    for (uint32_t h = 0; h < a.ngroups; ++h) {
                        const uint32_t c = *(volatile uint32_t*)&a.work[h];
                        if (c < a.nchunks && c < cmin) {
                            cmin = c;
                            gmin = h;
                        }
                    }
                    if (cmin == 0xFFFFFFFFu) break;
                    const uint32_t cg = *(volatile uint32_t*)&a.work[g];
                    if (cg >= a.nchunks || cg > cmin + POLY_AFFINE_LEAD) g = gmin;
                    const uint32_t c = atomicAdd(&a.work[g], 1u);
                    if (c < a.nchunks) {
                        u = c * a.ngroups + g;
                        break;
                    }
                }
                cg_s = g;
            } else {
                u = atomicAdd(a.work, 1u);
            }
            unit_s = u;
            dclaim_s = 0;
        }
        __syncthreads();
        const uint32_t unit = unit_s;
        if (unit >= a.units) break;
        const uint32_t g = unit % a.ngroups, chunk = unit / a.ngroups;
        const uint32_t q0 = g * Q;
        const uint32_t nqh = min((uint32_t)Q, a.nqb - q0);
        const uint64_t t0 = (uint64_t)chunk * a.tiles_per_chunk;
        const uint32_t ntile = (uint32_t)min((uint64_t)a.tiles_per_chunk, a.ntiles - t0);

        if (group_s != g) {  // the group's LUTs and the MMA's B operand (query weights + bias)
            const float4* src = reinterpret_cast<const float4*>(a.lutp + (size_t)q0 * M * KSUB);
            constexpr uint32_t PER_Q = M * KSUB / 4;
            for (uint32_t i = threadIdx.x; i < nqh * PER_Q; i += NT) {
                const uint32_t q = i / PER_Q, r = i % PER_Q;
                const float4 v = __ldg(src + i);
                float* d = lut + q * LS + 4 * r;
                d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
            }
            // B row n: element 8 (4 cw + s) + i = bit 32 cw + 4 i + s of query n -> +2 / -2 (e2m1 0x4 / 0xC);
            // K-major no swizzle, core (n8, k16) at n8 * 128 + k16 * 256
            if (threadIdx.x < 16 * 8) {
                const uint32_t n = threadIdx.x >> 3, wd = threadIdx.x & 7u, cw = wd >> 2, sh = wd & 3u;
                uint32_t v = 0x44444444u;
                if (n < nqh) v |= ((__ldg(reinterpret_cast<const uint32_t*>(a.qcodes) + (size_t)(q0 + n) * 2 + cw) >> sh) &
                                   0x11111111u) << 3;
                const uint32_t byte = wd * 4;
                *reinterpret_cast<uint32_t*>(bq_s + (n >> 3) * 128 + (byte >> 4) * 256 + (n & 7) * 16 + (byte & 15)) = v;
            }
            fence_proxy_async_smem();  // generic-proxy writes -> tensor-core reads
        }
        if (threadIdx.x < Q) {
            thr_s[threadIdx.x] = threadIdx.x < nqh ? __ldcg(a.thr + q0 + threadIdx.x) : 0ull;
            surv_s[threadIdx.x] = 0;
            if (PERQ) hash_s[threadIdx.x] = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) group_s = g;

        if (warp == PROD) {
            // ---------------------------------------------------------------- producer
            auto refresh = [&]() {  // keep the drains' bounds fresh (aligned 64-bit stores)
                if (lane < nqh) {
                    const unsigned long long t = __ldcg(a.thr + q0 + lane);
                    if (t < thr_s[lane]) thr_s[lane] = t;
                }
                __syncwarp();
            };
            for (uint32_t j = 0; j < ntile; ++j) {
                const uint32_t sq_ = seq + j, s = sq_ % STG;
                if (sq_ >= STG && lane == 0) mbar_wait(&empty_bar[s], ((sq_ / STG) - 1) & 1u);
                if (lane == 0) {
                    const uint64_t first = (t0 + j) * a.tile_stride * TC;
                    const uint64_t cnt = min((uint64_t)TC, a.n - first);
                    const uint32_t bytes = (uint32_t)((cnt * M + 15) & ~15ull);
                    mbar_arrive_expect_tx(&full_bar[s], bytes);
                    bulk_g2s(tiles + s * TC, a.codes + first * M, bytes, &full_bar[s]);
                }
                __syncwarp();
                serve_selects();
                refresh();
            }
        } else if (warp < NF) {
            // ---------------------------------------------------------------- filter
            const uint32_t quad = (uint32_t)warp >> 2, wq = (uint32_t)warp & 3u;
            const uint32_t row = 32 * wq + lane;  // this lane's A row / D lane within the quad
            // accumulator preload: D_q = |q| - tau - 1/2 (invalid queries: never pass)
            {
                const uint32_t tau = min(a.tau, (uint32_t)(M * 8));
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    float v = 1.0e6f;
                    if ((uint32_t)q < nqh) {
                        const uint2 qc = reinterpret_cast<const uint2*>(a.qcodes)[q0 + q];
                        v = (float)(__popc(qc.x) + __popc(qc.y)) - (float)tau - 0.5f;
                    }
                    bias[q] = v;
                }
            }
            const uint32_t a_smem = smem_u32(smem + AOFF);
            const uint64_t bdesc = (uint64_t)((smem_u32(bq_s) & 0x3FFFFu) >> 4) | ((uint64_t)(256u >> 4) << 16) |
                                   ((uint64_t)(128u >> 4) << 32) | (1ull << 46);
            const uint32_t nhalf = ntile * HSTEPS;
            // half-step hs of the unit (this quad's: hs = quad, quad + FQ, ...): tile hs / HSTEPS,
            // codes 128 (hs % HSTEPS) + [0, 128); this lane's code is 128 (hs % HSTEPS) + row,
            // i.e. slot 2 (hs % HSTEPS) + (row >= 64), lane bit half (row / 32) & 1
            auto where = [&](uint32_t hs, uint32_t& s, uint32_t& par, uint32_t& li, uint32_t& tcnt) {
                const uint32_t jt = hs / HSTEPS, sq_ = seq + jt;
                s = sq_ % STG;
                par = (sq_ / STG) & 1u;
                li = 128 * (hs % HSTEPS) + row;
                const uint64_t tfirst = (t0 + jt) * a.tile_stride * TC;
                tcnt = (uint32_t)min((uint64_t)TC, a.n - tfirst);
            };
            auto stage = [&](uint32_t hs, uint32_t b) {
                uint32_t s, par, li, tcnt;
                where(hs, s, par, li, tcnt);
                mbar_wait(&full_bar[s], par);
                C c;
                lds_code(tile_base + s * (uint32_t)TILE_BYTES + li * (uint32_t)M, c);
                // A row: element 8 (4 cw + sh) + i = bit 32 cw + 4 i + sh -> e2m1 0.5 (0x1) or 0;
                // K-major no swizzle, core (m8, k16) at m8 * 128 + k16 * 2048
                const uint32_t abuf = a_smem + (quad * NBUF + b) * A_BYTES;
                const uint32_t w0 = c.x & 0x11111111u, w1 = (c.x >> 1) & 0x11111111u, w2 = (c.x >> 2) & 0x11111111u,
                               w3 = (c.x >> 3) & 0x11111111u;
                const uint32_t w4 = c.y & 0x11111111u, w5 = (c.y >> 1) & 0x11111111u, w6 = (c.y >> 2) & 0x11111111u,
                               w7 = (c.y >> 3) & 0x11111111u;
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(abuf + row * 16), "r"(w0), "r"(w1),
                             "r"(w2), "r"(w3)
                             : "memory");
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(abuf + 2048 + row * 16), "r"(w4),
                             "r"(w5), "r"(w6), "r"(w7)
                             : "memory");
                fence_proxy_async_smem();  // generic-proxy A rows -> tensor-core reads
                tc_fence_before();
                named_bar_sync(1 + quad, 128);  // the quad's four warps staged their rows (uniform work)
                if (wq == 0 && lane == 0) {
                    tc_fence_after();
                    const uint64_t adesc = (uint64_t)(((a_smem + (quad * NBUF + b) * A_BYTES) & 0x3FFFFu) >> 4) |
                                           ((uint64_t)(2048u >> 4) << 16) | ((uint64_t)(128u >> 4) << 32) | (1ull << 46);
                    const uint32_t d_t = tbase + D_COL + 16u * (quad * NBUF + b);
#if POLY_K2T_DEBUG == 1
                    mbar_arrive(&qbar_s[quad * NBUF + b]);
#else
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.u32 p, 0, 0;\n"  // D = A.B (no accumulate)
                        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n}\n" ::"r"(
                            d_t),
                        "l"(adesc), "l"(bdesc), "r"(IDESC_MXF4_M128_N16), "r"(tbase + SF_COL), "r"(tbase + SF_COL + 16)
                        : "memory");
                    tc_commit(&qbar_s[quad * NBUF + b]);
#endif
                }
                __syncwarp();
            };
            auto finish = [&](uint32_t hs, uint32_t b, uint32_t gt) {  // gt: the warp's global count of hs
                uint32_t s, par, li, tcnt;
                where(hs, s, par, li, tcnt);
                mbar_wait(&qbar_s[quad * NBUF + b], (gt / NBUF) & 1u);
                tc_fence_after();
                uint32_t d[16], m = 0;
                tmem_ld16(tbase + tlane + D_COL + 16u * (quad * NBUF + b), d);
                tmem_wait_ld();
                // D_q = |x| - 2 <x, q>; + |q| - tau - 1/2 = h - tau - 1/2 (exact): sign bit = [h <= tau]
#pragma unroll
                for (int q = 15; q >= 0; --q) m = __funnelshift_l(__float_as_uint(__uint_as_float(d[q]) + bias[q]), m, 1);
                tc_fence_before();
                const uint32_t vm = (nqh >= 16 ? 0xFFFFu : (1u << nqh) - 1u);
                m &= li < tcnt ? vm : 0u;
                // lanes: code li = 128 h + 32 wq + lane; slot k = 2 h + (wq >> 1), its lane bit half = wq & 1
                // (slot k covers codes 64 k + lane and 64 k + lane + 32)
                // slot k = 2 (hs % HSTEPS) + (wq >> 1) gets its low / high 16 bits (codes 64 k + lane /
                // + 32) from warps wq even / odd of this quad; the slot's mbarrier counts both
                const uint32_t k = 2 * (hs % HSTEPS) + (wq >> 1);
                asm volatile("st.shared.u16 [%0], %1;" ::"r"(mask_base + 4u * ((s * NSLOT + k) * 32 + lane) +
                                                             2u * (wq & 1u)),
                             "h"((unsigned short)m)
                             : "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&slot_bar[s * NSLOT + k]);
            };
            uint32_t t = 0;  // half-steps of this unit
            for (uint32_t hs = quad; hs < nhalf; hs += FQ, ++t) {
                const uint32_t gt = fstep + t;
                stage(hs, gt % NBUF);
                if (t >= 1) finish(hs - FQ, (gt - 1) % NBUF, gt - 1);
            }
            if (t) finish(quad + (t - 1) * FQ, (fstep + t - 1) % NBUF, fstep + t - 1);
            fstep += t;
        } else {
            // ---------------------------------------------------------------- drain
            uint32_t* ring = rings + (warp - NF) * RING;
            const uint32_t ring_base = smem_u32(ring);
            uint32_t qn = 0, tot = 0;
            uint32_t survq[PERQ ? Q : 1];
#pragma unroll
            for (int q = 0; q < (PERQ ? Q : 1); ++q) survq[q] = 0;
            auto drain_at = [&](uint32_t T, uint64_t tfirst, uint32_t off, uint32_t cnt) {
                if ((uint32_t)lane < cnt) {
                    const uint32_t e = lds32v(ring_base + 4u * (off + lane));
                    const uint32_t pbit = e >> 16;  // bit p = 16 c + q
                    const uint32_t q = pbit & 15u;
                    const uint32_t li = (e & 0xFFFFu) + 32u * (pbit >> 4);
                    C code;
                    lds_code(T + li * (uint32_t)M, code);
                    const unsigned long long thr = thr_s[q];
                    if constexpr (PERQ)
                        atomicAdd(&hash_s[q], (unsigned long long)mix64(key_low(a, (uint32_t)(tfirst + li))));
                    const float score = adc_s_bounded<M>(lut_base + 4u * q * LS, code, (uint32_t)(thr >> 32));
                    try_candidate(a, q0 + q, score, (uint32_t)(tfirst + li), thr, bs, &nreq_s, req_s);
                }
            };
            auto drain_full = [&](uint32_t T, uint64_t tfirst) {
                uint32_t off = 0;
                while (qn - off >= 32) {
                    drain_at(T, tfirst, off, 32);
                    off += 32;
                }
                __syncwarp();
                if (off) {
                    const uint32_t rem = qn - off;
                    const uint32_t e = (uint32_t)lane < rem ? lds32v(ring_base + 4u * (off + lane)) : 0u;
                    __syncwarp();
                    if ((uint32_t)lane < rem) sts32(ring_base + 4u * lane, e);
                    qn = rem;
                }
                __syncwarp();
            };
            auto append = [&](uint32_t mm, uint32_t li, uint32_t excl) {
                uint32_t addr = ring_base + 4u * (qn + excl);
                while (mm) {
                    const uint32_t low = mm & (0u - mm);
                    sts32(addr, ((31u - __clz(low)) << 16) | li);
                    addr += 4;
                    mm ^= low;
                }
            };
            auto scan = [&](uint32_t cnt, uint32_t& total) {
                uint32_t incl = cnt;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += o;
                }
                total = __shfl_sync(0xffffffffu, incl, 31);
                return incl - cnt;
            };
            const uint32_t nslots = ntile * NSLOT;
            for (;;) {
                uint32_t d = 0;
                if (lane == 0) d = atomicAdd(&dclaim_s, 1u);
                d = __shfl_sync(0xffffffffu, d, 0);
                if (d >= nslots) break;
                const uint32_t jt = d / NSLOT, k = d % NSLOT, sq_ = seq + jt, s = sq_ % STG;
                mbar_wait(&slot_bar[s * NSLOT + k], (sq_ / STG) & 1u);
                const uint32_t m = lds32v(mask_base + 4u * ((s * NSLOT + k) * 32 + lane));
                const uint32_t T = tile_base + s * (uint32_t)TILE_BYTES;
                const uint64_t tfirst = (t0 + jt) * a.tile_stride * TC;
                const uint32_t li = k * 64 + lane;
                if constexpr (PERQ) {
#pragma unroll
                    for (int q = 0; q < Q; ++q)
                        survq[q] += __popc(__ballot_sync(0xffffffffu, (m >> q) & 1u)) +
                                    __popc(__ballot_sync(0xffffffffu, (m >> (q + 16)) & 1u));
                }
                if (__any_sync(0xffffffffu, m != 0)) {
                    uint32_t total;
                    const uint32_t excl = scan(__popc(m), total);
                    if (qn + total <= (uint32_t)RING) {
                        append(m, li, excl);
                        qn += total;
                        tot += total;
                        __syncwarp();
                        if (qn >= 32) drain_full(T, tfirst);
                    } else {
#pragma unroll 1
                        for (int part = 0; part < 32 / PART_BITS; ++part) {
                            const uint32_t mm = m & (((1u << PART_BITS) - 1u) << (PART_BITS * part));
                            uint32_t ptotal;
                            const uint32_t pex = scan(__popc(mm), ptotal);
                            append(mm, li, pex);
                            qn += ptotal;
                            tot += ptotal;
                            __syncwarp();
                            if (qn >= 32) drain_full(T, tfirst);
                        }
                    }
                }
                if (qn) {  // entries point into this stage: flush before the release
                    drain_at(T, tfirst, 0, qn);
                    qn = 0;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);
            }
            if (lane == 0) {
                if constexpr (PERQ) {
                    for (int q = 0; q < Q; ++q)
                        if (survq[q]) atomicAdd(&surv_s[q], survq[q]);
                } else if (tot) {
                    atomicAdd(&surv_s[0], tot);
                }
            }
        }
        seq += ntile;
        __syncthreads();
        if (warp == PROD) serve_selects();  // blocks completed during the unit's last tiles
        if (threadIdx.x < (PERQ ? nqh : 1u) && surv_s[threadIdx.x]) {
            atomicAdd(a.surv + (PERQ ? q0 + threadIdx.x : 0u), (unsigned long long)surv_s[threadIdx.x]);
            if (PERQ) atomicAdd(a.surv_hash + q0 + threadIdx.x, hash_s[threadIdx.x]);
        }
        __syncthreads();
    }
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tbase, 128);
}

void launch_scan_tc(const ScanArgs& a, bool per_query_stats, int num_sms, cudaStream_t s) {
    const size_t smem = k2t::TOTAL;
    auto kfn = per_query_stats ? scan_tc_kernel<true> : scan_tc_kernel<false>;
    set_max_smem((const void*)kfn, smem);
    const unsigned grid = (unsigned)((uint64_t)num_sms < (uint64_t)a.units ? (uint64_t)num_sms : (uint64_t)a.units);
    kfn<<<grid, k2t::NW * 32, smem, s>>>(a);
    count_launch();
}

}  // namespace pb
