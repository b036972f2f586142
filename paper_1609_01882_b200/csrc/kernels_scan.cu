// kernels_scan.cu -- K2: fused Hamming filter + ADC + candidate scan (sm_100a).
//
// One pass over the database per query group replaces the reference's two
// passes (restated in the oracle):
//   hamming_bytes   flat_index.hpp:14-27   popc(qcode ^ code), kept iff h <= tau
//   adc_distance    pq.cpp:121-128         acc = 0; acc += LUTp[sq][field_sq] in sq order
//   TopK::offer     flat_index.hpp:64-76   replaced by a key-threshold candidate append; the
//                                          exact top-k is taken by K3 (kernels_topk.cu)
//
// CTA = W consumer warps + 1 TMA producer warp.  Work unit = (chunk of tiles,
// group of Q queries), fetched dynamically.  The producer streams 16 KB code
// tiles HBM -> shared memory through a STAGES-deep ring of 1-D bulk copies
// (cp.async.bulk + mbarrier complete_tx) and recycles a stage once all W
// consumer warps have arrived on its "empty" mbarrier -- no CTA-wide barrier
// per tile.  Each consumer lane holds one code in registers and tests it
// against the Q query codes branch-free (xor + 2 POPC + compare per pair),
// building a per-lane survivor mask; a warp prefix scan compacts survivors
// into a per-warp ring of 4-byte entries (query | tile index).  Whenever 32
// entries are queued the warp drains them with all lanes busy: the code is
// re-read from the tile, 8/16 gathers from the query's stored-field LUT in
// shared memory are summed in sub-quantizer order with __fadd_rn (bit-exact
// with the reference), and the key is tested against the query's threshold.
//
// Candidates: key = (fp32 score bits << 32) | id-rank (scores are >= 0 so the
// bits are monotone; ranks are distinct) -- a strict total order equal to the
// SPEC (score, id) order.  A candidate is appended to its query's global list
// when key < thr[q].  thr[q] is an upper bound of the final k-th key: whenever
// a block of BS consecutive list slots completes, the producer warp of the
// CTA that completed it selects the block's k-th smallest key (radix select)
// and atomicMin's it into thr[q].  thr[] starts from the exact k-th key of
// strided warm-up samples (capi.cu), so these selects are rare.  Every final
// top-k member is in the list; K3 takes the exact top-k.
#include "scan_common.cuh"

namespace pb {

#ifndef POLY_TC  // 1: DUAL's Hamming filter on the tensor cores (int8 tcgen05.mma); 0: POPC
#define POLY_TC 1
#endif
#ifndef POLY_RING
#define POLY_RING 288
#endif
// per-warp survivor queue (4-byte entries, linear): < 32 left + one step part;
// a step that does not fit is split into mask parts of PART_BITS bits (<= 32 * PART_BITS entries)
constexpr int RING = POLY_RING;
constexpr int PART_BITS = RING >= 32 + 256 ? 8 : 4;

template <int M, int Q, int W>
struct ScanSmem {
    static constexpr int TC = TILE_BYTES / M;               // codes per tile
    // Query q's LUT starts at q * LS floats; the +1 skew puts the same stored
    // field of up to 32 different queries in different banks (a drain holds
    // many queries' entries for the same code).
    static constexpr int LS = M * KSUB + 1;
    static constexpr size_t LUT_BYTES = (size_t)Q * LS * 4;
    static constexpr size_t TILES = (size_t)STAGES * TILE_BYTES;
    static constexpr size_t RING_BYTES = (size_t)W * RING * 4;
    static constexpr size_t TOTAL = LUT_BYTES + TILES + RING_BYTES;
};

// PERQ: per-query survivor counts (ballot + popc per query) instead of the
// free per-batch total.
template <int M, int Q, int W, int STRAT, bool PERQ>
__global__ void __launch_bounds__((W + 1) * 32, 1) scan_kernel(const ScanArgs a) {
    static_assert(RING >= 32 + 32 * PART_BITS, "ring must hold a remainder plus one mask part");
    const uint32_t bs = a.bs;
    using C = typename CodeT<M>::T;
    using SM = ScanSmem<M, Q, W>;
    constexpr int NT = (W + 1) * 32;
    constexpr int TC = SM::TC;
    constexpr int CPW = TC / W;     // codes per consumer warp per tile
    constexpr bool USE_LUT = (STRAT == DUAL || STRAT == ADC);
    static_assert(CPW % 64 == 0, "tile must split evenly over the consumer warps (2 codes per lane per step)");

    extern __shared__ __align__(128) uint8_t smem[];
    float* lut = reinterpret_cast<float*>(smem);
    C* tiles = reinterpret_cast<C*>(smem + (USE_LUT ? SM::LUT_BYTES : 0));
    uint32_t* rings = reinterpret_cast<uint32_t*>(smem + (USE_LUT ? SM::LUT_BYTES : 0) + SM::TILES);

    __shared__ __align__(8) uint64_t full_bar[STAGES];
    __shared__ __align__(8) uint64_t empty_bar[STAGES];
    __shared__ unsigned long long thr_s[Q];
    __shared__ C qc_s[Q];
    __shared__ uint32_t surv_s[Q];
    __shared__ unsigned long long hash_s[PERQ ? Q : 1];
    __shared__ uint32_t unit_s, nreq_s, group_s;
    __shared__ uint32_t req_s[MAXREQ];
    __shared__ uint32_t sel_hist[256];
    __shared__ uint32_t req_head_s;
    // tensor-core filter state: B operand (query weights + bias), per-quad MMA barriers, TMEM base
    // m = 16 keeps the POPC filter: 8 queries per CTA do not amortise the bit-plane expansion
    // (A/B in DESIGN.md sec. 5)
    constexpr bool TCF = POLY_TC && STRAT == DUAL && M == 8;
    constexpr int KB = M * 8 + 32;   // B row bytes: one per code bit + the bias block
    constexpr int NKB = KB / 32;     // K blocks of 32 bytes
    constexpr int AC = 2 * M;        // TMEM columns of one expanded code (M * 8 bytes)
    constexpr int QC = 2 * AC + 32;  // columns per quad: A0, A1, D0, D1
    static_assert(!TCF || (W % 4 == 0 && 16 + (W / 4) * QC <= 512), "TMEM budget");
    __shared__ __align__(256) int8_t bw_s[TCF ? 16 * KB : 16];
    __shared__ __align__(8) uint64_t qbar_s[W / 4];
    __shared__ uint32_t qcnt_s[W / 4];  // A-row stagings per quad (the 4th of each round issues the MMA)
    __shared__ uint32_t tmem_s;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = warp == W;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], W);
        }
        fence_mbar_init();
        if (TCF)
            for (int qd = 0; qd < W / 4; ++qd) {
                mbar_init(&qbar_s[qd], 1);
                qcnt_s[qd] = 0;
            }
        fence_mbar_init();
        nreq_s = 0;
        req_head_s = 0;
        group_s = 0xFFFFFFFFu;
    }
    if (threadIdx.x < MAXREQ) req_s[threadIdx.x] = 0xFFFFFFFFu;
    if (TCF && warp == 0) tmem_alloc(&tmem_s, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = TCF ? tmem_s : 0u;
    // TMEM: columns [0, 8) = the A bias block (constant 2), quad k at 16 + k * QC
    const uint32_t tlane = (uint32_t)(32 * (warp & 3)) << 16;
    if (TCF && warp < 4) {
        tmem_st8(tbase + tlane, 0x02020202u);
        tmem_wait_st();
    }
    tc_fence_before();

    uint32_t* ring = rings + (producer ? 0 : warp) * RING;
    uint32_t seq = 0;
    uint32_t qphase = 0;  // parity of this warp's quad MMA barrier

    // producer warp: serve threshold selects requested by the consumers' appends
    auto serve_selects = [&]() {
        for (;;) {
            uint32_t req = 0xFFFFFFFFu;
            if (lane == 0) {
                const uint32_t tail = *(volatile uint32_t*)&nreq_s;
                if (tail - req_head_s > MAXREQ) req_head_s = tail - MAXREQ;  // dropped requests
                if (req_head_s != tail) {
                    // the writer moves the tail before it fills the slot: EMPTY = not yet published
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
            if (qg >= a.nqb || blk >= a.cap / bs) continue;  // (a lapped slot still holds some valid request)
            __threadfence();
            const unsigned long long kth =
                warp_select_kth(a.cand + (size_t)qg * a.cap + (size_t)blk * bs, bs, a.k, sel_hist);
            if (lane == 0) atomicMin(a.thr + qg, kth);
        }
    };  // tiles consumed so far: stage = seq % STAGES, parity = (seq / STAGES) & 1

    __shared__ uint32_t cg_s;  // affine schedule: this CTA's current query group
    if (threadIdx.x == 0) cg_s = blockIdx.x % a.ngroups;
    for (;;) {
        if (threadIdx.x == 0) {
            if (a.affine) {
                // next chunk of the current group.  A group may lead the slowest group
                // still holding work by at most POLY_AFFINE_LEAD chunks: beyond that (or when
                // its own group is dry) the CTA helps the slowest group (one LUT reload).  All
                // groups then sweep the same window of the database, which L2 keeps, so
                // the codes are read from HBM about once per batch.
                uint32_t g = cg_s, u = a.units;
                for (uint32_t tries = 0; tries < 4 * a.ngroups + 4; ++tries) {
                    uint32_t gmin = g, cmin = 0xFFFFFFFFu;
                    for (uint32_t h = 0; h < a.ngroups; ++h) {
                        const uint32_t c = *(volatile uint32_t*)&a.work[h];
                        if (c < a.nchunks && c < cmin) {
                            cmin = c;
                            gmin = h;
                        }
                    }
                    if (cmin == 0xFFFFFFFFu) break;  // every group is dry
                    const uint32_t cg = *(volatile uint32_t*)&a.work[g];
                    if (cg >= a.nchunks || cg > cmin + POLY_AFFINE_LEAD) g = gmin;
                    const uint32_t c = atomicAdd(&a.work[g], 1u);
                    if (c < a.nchunks) {
                        u = c * a.ngroups + g;
                        break;
                    }
                }
                cg_s = g;
                unit_s = u;
            } else {
                unit_s = atomicAdd(a.work, 1u);
            }
        }
        __syncthreads();
        const uint32_t unit = unit_s;
        if (unit >= a.units) break;
        const uint32_t g = unit % a.ngroups, chunk = unit / a.ngroups;
        const uint32_t q0 = g * Q;
        const uint32_t nqh = min((uint32_t)Q, a.nqb - q0);
        const uint64_t t0 = (uint64_t)chunk * a.tiles_per_chunk;
        const uint32_t ntile = (uint32_t)min((uint64_t)a.tiles_per_chunk, a.ntiles - t0);

        // per-group state: LUTs (only when the group changes), query codes, thresholds
        if (group_s != g) {
            if (USE_LUT) {
                const float4* src = reinterpret_cast<const float4*>(a.lutp + (size_t)q0 * M * KSUB);
                constexpr uint32_t PER_Q = M * KSUB / 4;
                const uint32_t n4 = nqh * PER_Q;
                for (uint32_t i = threadIdx.x; i < n4; i += NT) {
                    const uint32_t q = i / PER_Q, r = i % PER_Q;
                    const float4 v = __ldg(src + i);
                    float* d = lut + q * SM::LS + 4 * r;  // rows are not 16-byte aligned
                    d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
                }
            }
            if (threadIdx.x < Q)
                qc_s[threadIdx.x] = threadIdx.x < nqh ? reinterpret_cast<const C*>(a.qcodes)[q0 + threadIdx.x] : C{};
            if (TCF) {
                const uint32_t* qw = reinterpret_cast<const uint32_t*>(a.qcodes);
                const uint32_t tau = min(a.tau, (uint32_t)(M * 8));
                for (uint32_t i = threadIdx.x; i < 16u * KB; i += NT) {
                    const uint32_t n = i / KB, k = i % KB;
                    int v = 0;
                    if (n < nqh) {
                        const uint32_t* qn = qw + (size_t)(q0 + n) * (M / 4);
                        if (k < (uint32_t)M * 8) {  // word k/32, plane j, byte t -> bit 8t + j
                            const uint32_t j = (k & 31u) >> 2, t = k & 3u;
                            const int mag = j < 7 ? (1 << (6 - j)) : 64;
                            v = ((__ldg(qn + (k >> 5)) >> (8 * t + j)) & 1u) ? -mag : mag;
                        } else {  // bias: 32 entries summing to 32 (|q| - tau) - 16
                            int pc = 0;
                            for (int w = 0; w < M / 4; ++w) pc += __popc(__ldg(qn + w));
                            const int T = 32 * (pc - (int)tau) - 16, e = (int)(k - (uint32_t)M * 8);
                            const int base = T / 32, rem = T - base * 32;
                            v = base + (e < (rem < 0 ? -rem : rem) ? (rem < 0 ? -1 : 1) : 0);
                        }
                    }
                    bw_s[bw_offset(n, k)] = (int8_t)v;
                }
                fence_proxy_async_smem();  // generic-proxy writes -> tensor-core reads
            }
        }
        if (threadIdx.x < Q) {
            thr_s[threadIdx.x] = threadIdx.x < nqh ? __ldcg(a.thr + q0 + threadIdx.x) : 0ull;
            surv_s[threadIdx.x] = 0;
            if (PERQ) hash_s[threadIdx.x] = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) group_s = g;

        if (producer) {
            // keep the consumers' thresholds fresh (benign race: aligned 64-bit stores)
            auto refresh = [&]() {
                if (lane < nqh) {
                    const unsigned long long t = __ldcg(a.thr + q0 + lane);
                    if (t < thr_s[lane]) thr_s[lane] = t;
                }
                __syncwarp();
            };
            for (uint32_t j = 0; j < ntile; ++j) {
                const uint32_t sq_ = seq + j, s = sq_ % STAGES;
                if (sq_ >= STAGES && lane == 0) mbar_wait(&empty_bar[s], ((sq_ / STAGES) - 1) & 1u);
                if (lane == 0) {
                    const uint64_t first = (t0 + j) * a.tile_stride * TC;
                    const uint64_t cnt = min((uint64_t)TC, a.n - first);
                    const uint32_t bytes = (uint32_t)((cnt * M + 15) & ~15ull);
                    mbar_arrive_expect_tx(&full_bar[s], bytes);
                    bulk_g2s(tiles + s * TC, a.codes + first * M, bytes, &full_bar[s]);
                }
                serve_selects();
                refresh();
            }
        } else {
            const C* qc = qc_s;  // query codes read from shared memory (broadcast): frees 2Q registers
            // survivor mask layout: query q = 4g + j -> bit 8j + g (g < Q/4, j < 4)
            uint32_t vmask = 0;
            for (uint32_t q = 0; q < nqh; ++q) vmask |= 1u << (8 * (q & 3) + (q >> 2));
            // h <= tau  <=>  bit 7 of (h + 127 - tau) clear, four bytes at a time
            const uint32_t bias = (127u - min(a.tau, 127u)) * 0x01010101u;
            const uint32_t lut_base = smem_u32(lut);
            const uint32_t tile_base = smem_u32(tiles);
            const uint32_t ring_base = smem_u32(ring);
            uint32_t qn = 0;   // queued survivor entries: ring[0, qn)
            uint32_t tot = 0;  // survivors seen by this warp (warp-uniform)
            uint32_t survq[PERQ ? Q : 1];
#pragma unroll
            for (int q = 0; q < (PERQ ? Q : 1); ++q) survq[q] = 0;

            // ADC + candidate test of `cnt` queued survivors starting at ring[off]
            // (lanes < cnt busy)
            auto drain_at = [&](uint32_t T, uint64_t tfirst, uint32_t off, uint32_t cnt) {
                if ((uint32_t)lane < cnt) {
                    const uint32_t e = lds32v(ring_base + 4u * (off + lane));
                    // mask bit p = 8j + 4c + g -> query 4g + j of the lane's code c (tile index li + 32c)
                    const uint32_t pbit = e >> 16;
                    // TCF: bit p = 16c + q; POPC: p = 8j + 4c + g for query 4g + j
                    const uint32_t q = TCF ? (pbit & 15u) : 4 * (pbit & 3) + (pbit >> 3);
                    const uint32_t li = (e & 0xFFFFu) + 32u * (TCF ? (pbit >> 4) : ((pbit >> 2) & 1u));
                    C code;
                    lds_code(T + li * (uint32_t)M, code);
                    const unsigned long long thr = thr_s[q];
                    if constexpr (PERQ)  // every queued entry is a filter survivor
                        atomicAdd(&hash_s[q], (unsigned long long)mix64(key_low(a, (uint32_t)(tfirst + li))));
                    const float score = adc_s_bounded<M>(lut_base + 4u * q * SM::LS, code, (uint32_t)(thr >> 32));
                    try_candidate(a, q0 + q, score, (uint32_t)(tfirst + li), thr, bs, &nreq_s, req_s);
                }
            };
            // drain full groups of 32, then move the (< 32) remainder to the front
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
            // append the lanes' survivor bits (entry = bit position << 16 | tile index)
            auto append = [&](uint32_t mm, uint32_t li, uint32_t excl) {
                uint32_t addr = ring_base + 4u * (qn + excl);
                const uint32_t lo = li;
                while (mm) {
                    const uint32_t low = mm & (0u - mm);
                    sts32(addr, ((31u - __clz(low)) << 16) | lo);
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

            // TCF: tile j's A rows (expanded codes) are staged into TMEM one tile ahead;
            // the quad's last warp to stage issues the MMA (no quad barrier)
            const uint32_t quad = (uint32_t)warp >> 2;
            const uint32_t A0 = tbase + tlane + 16u + quad * QC, A1 = A0 + AC;
            const uint32_t D0 = A0 + 2 * AC, D1 = D0 + 16;
            const uint32_t qa0 = tbase + 16u + quad * QC;   // lane 0 of the quad's columns
            const uint64_t bdesc0 = bw_desc(smem_u32(bw_s));  // + 32 per K block (512 B >> 4)
            auto stage_a = [&](uint32_t jj) {
                const uint32_t sq_ = seq + jj, s = sq_ % STAGES;
                mbar_wait_backoff(&full_bar[s], (sq_ / STAGES) & 1u);
                const uint32_t T = tile_base + s * (uint32_t)TILE_BYTES;
                const uint32_t li = warp * CPW + lane;
                C c0, c1;
                lds_code(T + li * (uint32_t)M, c0);
                lds_code(T + (li + 32) * (uint32_t)M, c1);
                uint32_t x[16];
#pragma unroll
                for (int h = 0; h < M / 8; ++h) {
                    expand_word(word(c0, 2 * h), x);
                    expand_word(word(c0, 2 * h + 1), x + 8);
                    tmem_st16(A0 + 16 * h, x);
                }
#pragma unroll
                for (int h = 0; h < M / 8; ++h) {
                    expand_word(word(c1, 2 * h), x);
                    expand_word(word(c1, 2 * h + 1), x + 8);
                    tmem_st16(A1 + 16 * h, x);
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0 && (atom_add_acq_rel(&qcnt_s[quad], 1u) & 3u) == 3u) {
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const uint32_t ac = qa0 + c * AC, dc = qa0 + 2 * AC + 16 * c;
#pragma unroll
                        for (int kb = 0; kb < NKB - 1; ++kb)
                            mma_i8_ts(dc, ac + 8 * kb, bdesc0 + (uint64_t)(32 * kb), IDESC_I8_M128_N16, kb);
                        mma_i8_ts(dc, tbase, bdesc0 + (uint64_t)(32 * (NKB - 1)), IDESC_I8_M128_N16, 1);
                    }
                    tc_commit(&qbar_s[quad]);
                }
                __syncwarp();
            };
            if constexpr (TCF) stage_a(0);
            for (uint32_t j = 0; j < ntile; ++j) {
                const uint32_t sq_ = seq + j, s = sq_ % STAGES;
                if constexpr (!TCF) mbar_wait_backoff(&full_bar[s], (sq_ / STAGES) & 1u);
                const uint32_t T = tile_base + s * (uint32_t)TILE_BYTES;
                const uint64_t tfirst = (t0 + j) * a.tile_stride * TC;
                const uint32_t tcnt = (uint32_t)min((uint64_t)TC, a.n - tfirst);
                if constexpr (STRAT == DUAL) {
                    // two codes per lane per step (li, li + 32): independent filter chains
#pragma unroll 1
                    for (int i = 0; i < CPW / 64; ++i) {
                        const uint32_t li = warp * CPW + i * 64 + lane;
                        uint32_t m;
                        if constexpr (TCF) {
                            // this tile's MMA was issued when the quad's last warp staged it
                            mbar_wait_backoff<POLY_SPIN_MMA_NS>(&qbar_s[quad], qphase);
                            qphase ^= 1u;
                            tc_fence_after();
                            // sign bits: bit q <- code li, bit 16 + q <- code li + 32
                            uint32_t d[16];
                            m = 0;
                            tmem_ld16(D1, d);
                            tmem_wait_ld();
#pragma unroll
                            for (int q = 15; q >= 0; --q) m = __funnelshift_l(d[q], m, 1);
                            tmem_ld16(D0, d);
                            tmem_wait_ld();
#pragma unroll
                            for (int q = 15; q >= 0; --q) m = __funnelshift_l(d[q], m, 1);
                            const uint32_t vm = (nqh >= 16 ? 0xFFFFu : (1u << nqh) - 1u);
                            m &= (li < tcnt ? vm : 0u) | (li + 32 < tcnt ? vm << 16 : 0u);
                            // stage the next tile's A rows now: its MMA overlaps this tile's survivors
                            if (j + 1 < ntile) stage_a(j + 1);
                        } else {
                            C c0, c1;
                            lds_code(T + li * (uint32_t)M, c0);
                            lds_code(T + (li + 32) * (uint32_t)M, c1);
                            uint32_t m0 = 0, m1 = 0;
#pragma unroll
                            for (int g = 0; g < Q / 4; ++g) {
                                const uint32_t v0 = ham4(c0, qc + 4 * g) + bias;
                                const uint32_t v1 = ham4(c1, qc + 4 * g) + bias;
                                m0 |= (~v0 & 0x80808080u) >> (7 - g);
                                m1 |= (~v1 & 0x80808080u) >> (3 - g);
                            }
                            m = (li < tcnt ? m0 & vmask : 0u) | (li + 32 < tcnt ? m1 & (vmask << 4) : 0u);
                        }
                        if constexpr (PERQ) {
#pragma unroll
                            for (int q = 0; q < Q; ++q) {
                                const int b = TCF ? q : 8 * (q & 3) + (q >> 2), b2 = TCF ? q + 16 : b + 4;
                                survq[q] += __popc(__ballot_sync(0xffffffffu, (m >> b) & 1u)) +
                                            __popc(__ballot_sync(0xffffffffu, (m >> b2) & 1u));
                            }
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
                                // a step adds <= 64 * Q entries: split it by mask part
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
                    }
                } else {
#pragma unroll 1
                    for (int i = 0; i < CPW / 32; ++i) {
                        const uint32_t li = warp * CPW + i * 32 + lane;
                        C code;
                        lds_code(T + li * (uint32_t)M, code);
                        // adc / binary / disidx: every code is scored for every query
                        if (li < tcnt) {
#pragma unroll 1
                            for (int q = 0; q < (int)nqh; ++q) {
                                float score;
                                if constexpr (STRAT == ADC)
                                    score = adc_s_bounded<M>(lut_base + 4u * q * SM::LS, code,
                                                             (uint32_t)(thr_s[q] >> 32));
                                else if constexpr (STRAT == BINARY) score = (float)ham(code, qc[q]);
                                else score = (float)disidx(code, qc[q]);
                                try_candidate(a, q0 + q, score, (uint32_t)(tfirst + li), thr_s[q], bs, &nreq_s,
                                              req_s);
                            }
                        }
                    }
                }
                if constexpr (STRAT == DUAL) {
                    if (qn) {  // entries point into this stage: flush before release
                        drain_at(T, tfirst, 0, qn);
                        qn = 0;
                        __syncwarp();
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);
            }
            if (STRAT == DUAL && lane == 0) {
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
        if (producer) serve_selects();  // blocks completed during the unit's last tiles
        // unit boundary: survivor stats flush
        // per-query counts -> surv[q]; totals -> surv[0] (the batch total)
        if (STRAT == DUAL && threadIdx.x < (PERQ ? nqh : 1u) && surv_s[threadIdx.x]) {
            atomicAdd(a.surv + (PERQ ? q0 + threadIdx.x : 0u), (unsigned long long)surv_s[threadIdx.x]);
            if (PERQ) atomicAdd(a.surv_hash + q0 + threadIdx.x, hash_s[threadIdx.x]);
        }
        __syncthreads();
    }
    if (TCF) {
        tc_fence_after();
        if (warp == 0) tmem_dealloc(tbase, 512);
    }
}

// K2s: threshold seed from a fixed sample, one CTA per query.  The sample is
// seed_blocks <= n / 256 disjoint runs of 256 consecutive codes spread evenly over the database
// (coalesced loads; the same runs for every query, so they stay in L2).  Each
// sampled code is scored exactly as K2 does (filter, then ADC / Hamming /
// disidx); the k-th smallest key of the sample (8-pass radix select over the
// keys staged in shared memory) bounds the final k-th key, so
// thr[q] = min(thr[q], kth + 1).  A key buffer that fills up keeps the first
// SEED_KEYS keys: the k-th of a subset is a weaker but still valid bound.
#ifndef POLY_SEED_KEYS
#define POLY_SEED_KEYS 4096
#endif
constexpr uint32_t SEED_THREADS = 256, SEED_KEYS = POLY_SEED_KEYS;

template <int M, int STRAT>
__global__ void __launch_bounds__(SEED_THREADS) seed_sample_kernel(const ScanArgs a, uint32_t seed_blocks) {
    using C = typename CodeT<M>::T;
    extern __shared__ __align__(16) uint8_t sm[];
    float* lut = reinterpret_cast<float*>(sm);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(sm + M * KSUB * 4);
    __shared__ uint32_t cnt, hist[256];
    __shared__ unsigned long long prefix_s;
    __shared__ uint32_t want_s;
    const uint32_t q = blockIdx.x;
    constexpr bool USE_LUT = (STRAT == DUAL || STRAT == ADC);
    if (USE_LUT)
        for (uint32_t i = threadIdx.x; i < (uint32_t)M * KSUB; i += SEED_THREADS)
            lut[i] = __ldg(a.lutp + (size_t)q * M * KSUB + i);
    const C qc = reinterpret_cast<const C*>(a.qcodes)[q];
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    constexpr uint32_t SU = 8;  // runs per step: their loads are in flight together
    for (uint32_t b0 = 0; b0 < seed_blocks; b0 += SU) {
        C codes_u[SU];
        uint64_t pos_u[SU];
#pragma unroll
        for (uint32_t u = 0; u < SU; ++u) {
            pos_u[u] = b0 + u < seed_blocks ? (uint64_t)(b0 + u) * a.n / seed_blocks + threadIdx.x : a.n;
            if (pos_u[u] < a.n) codes_u[u] = __ldg(reinterpret_cast<const C*>(a.codes) + pos_u[u]);
        }
#pragma unroll
        for (uint32_t u = 0; u < SU; ++u) {
            const uint64_t pos = pos_u[u];
            if (pos >= a.n) continue;
            const C code = codes_u[u];
            float score;
            if constexpr (STRAT == DUAL) {
                if (ham(code, qc) > a.tau) continue;
                score = adc<M>(lut, code);
            } else if constexpr (STRAT == ADC) {
                score = adc<M>(lut, code);
            } else if constexpr (STRAT == BINARY) {
                score = (float)ham(code, qc);
            } else {
                score = (float)disidx(code, qc);
            }
            const uint32_t slot = atomicAdd(&cnt, 1u);
            if (slot < SEED_KEYS)
                keys[slot] = ((unsigned long long)__float_as_uint(score) << 32) | key_low(a, (uint32_t)pos);
        }
    }
    __syncthreads();
    const uint32_t n = min(cnt, SEED_KEYS);
    if (n < a.k) return;  // too few keys in the sample: no bound
    unsigned long long prefix = 0, mask = 0;
    uint32_t want = a.k;
    for (int shift = 56; shift >= 0; shift -= 8) {
        hist[threadIdx.x] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += SEED_THREADS) {
            const unsigned long long v = keys[i];
            if ((v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 0xFFu], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const uint32_t lane = threadIdx.x;
            uint32_t c[8], t = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) { c[j] = hist[lane * 8 + j]; t += c[j]; }
            uint32_t incl = t;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += o;
            }
            const uint32_t excl = incl - t;
            if (excl < want && want <= incl) {
                uint32_t r = want - excl;
                int digit = lane * 8 + 7;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (r <= c[j]) { digit = lane * 8 + j; break; }
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
static void launch_seed_m(const ScanArgs& a, uint32_t nq, uint32_t seed_blocks, cudaStream_t s) {
    const size_t smem = (size_t)M * KSUB * 4 + SEED_KEYS * 8;
    auto kfn = seed_sample_kernel<M, STRAT>;
    set_max_smem((const void*)kfn, smem);
    kfn<<<nq, SEED_THREADS, smem, s>>>(a, seed_blocks);
    count_launch();
}

void launch_seed_sample(const ScanArgs& a, int strategy, uint32_t m, uint32_t nq, uint32_t seed_blocks,
                        cudaStream_t s) {
    if (nq == 0 || seed_blocks == 0) return;
    const bool w = m == 16;
    switch (strategy) {
        case DUAL: w ? launch_seed_m<16, DUAL>(a, nq, seed_blocks, s) : launch_seed_m<8, DUAL>(a, nq, seed_blocks, s); break;
        case ADC: w ? launch_seed_m<16, ADC>(a, nq, seed_blocks, s) : launch_seed_m<8, ADC>(a, nq, seed_blocks, s); break;
        case BINARY:
            w ? launch_seed_m<16, BINARY>(a, nq, seed_blocks, s) : launch_seed_m<8, BINARY>(a, nq, seed_blocks, s);
            break;
        default:
            w ? launch_seed_m<16, DISIDX>(a, nq, seed_blocks, s) : launch_seed_m<8, DISIDX>(a, nq, seed_blocks, s);
            break;
    }
}

template <int M, int Q, int W, int STRAT, bool PERQ>
static void launch_one(const ScanArgs& a, int num_sms, cudaStream_t s) {
    using SM = ScanSmem<M, Q, W>;
    constexpr bool USE_LUT = (STRAT == DUAL || STRAT == ADC);
    const size_t smem = USE_LUT ? SM::TOTAL : SM::TOTAL - SM::LUT_BYTES;
    auto kfn = scan_kernel<M, Q, W, STRAT, PERQ>;
    set_max_smem((const void*)kfn, smem);
    const unsigned grid = (unsigned)((uint64_t)num_sms < (uint64_t)a.units ? (uint64_t)num_sms : (uint64_t)a.units);
    kfn<<<grid, (W + 1) * 32, smem, s>>>(a);
    count_launch();
}

int scan_queries_per_cta(uint32_t m) { return m == 8 ? 16 : 8; }

template <int M, int Q, int W>
static void launch_m(const ScanArgs& a, int strategy, bool perq, int num_sms, cudaStream_t s) {
    switch (strategy) {
        case DUAL:
            if (perq) launch_one<M, Q, W, DUAL, true>(a, num_sms, s);
            else launch_one<M, Q, W, DUAL, false>(a, num_sms, s);
            break;
        case ADC: launch_one<M, Q, W, ADC, false>(a, num_sms, s); break;
        case BINARY: launch_one<M, Q, W, BINARY, false>(a, num_sms, s); break;
        default: launch_one<M, Q, W, DISIDX, false>(a, num_sms, s); break;
    }
}

void launch_scan(const ScanArgs& a, int strategy, uint32_t m, bool per_query_stats, int num_sms, cudaStream_t s) {
    // Q queries per CTA: Q x m x 1 KB of LUTs must fit next to the tile ring.
    if (m == 8) launch_m<8, 16, SCAN_WARPS>(a, strategy, per_query_stats, num_sms, s);
    else launch_m<16, 8, SCAN_WARPS / 2>(a, strategy, per_query_stats, num_sms, s);
}

}  // namespace pb
