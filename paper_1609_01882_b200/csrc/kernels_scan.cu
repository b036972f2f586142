// kernels_scan.cu -- K2: fused Hamming filter + ADC + candidate scan (sm_100a).
//
// One pass over the database per query group replaces the reference's two
// passes (SPEC.md:336 restated in the oracle):
//   hamming_bytes   flat_index.hpp:14-27   popc(qcode ^ code), kept iff h <= tau
//   adc_distance    pq.cpp:121-128         acc = 0; acc += LUTp[sq][field_sq] in sq order
//   TopK::offer     flat_index.hpp:64-76   replaced by key-threshold candidate append; the
//                                          exact top-k is taken by K3 (kernels_topk.cu)
//
// Work unit = (chunk of tiles, group of Q queries).  A CTA owns one unit at a
// time (dynamic fetch).  Code tiles stream HBM -> shared memory through a
// 4-deep ring of 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx).
// Each lane holds one code in registers and tests it against the Q query
// codes; survivors are compacted with a warp ballot into a per-warp queue
// (code + position + query).  Whenever 32 entries are queued the warp drains
// them with all lanes busy: 8/16 gathers from the query's stored-field LUT in
// shared memory, summed in sub-quantizer order with __fadd_rn (bit-exact).
//
// Candidates: key = (fp32 score bits << 32) | id-rank (scores are >= 0 so the
// bits are monotone; ranks are distinct) -- a strict total order equal to the
// SPEC (score, id) order.  A candidate is appended to its query's global list
// when key < thr[q].  thr[q] is an upper bound of the final k-th key: whenever
// a block of BS consecutive list slots completes, the CTA that completed it
// selects the block's k-th smallest key (radix select) and atomicMin's it
// into thr[q].  Every final top-k member is therefore in the list.
#include "poly_b200.cuh"

namespace pb {

template <int M> struct CodeT;
template <> struct CodeT<8> { using T = uint2; };
template <> struct CodeT<16> { using T = uint4; };

__device__ __forceinline__ uint32_t ham(const uint2& a, const uint2& b) {
    return __popc(a.x ^ b.x) + __popc(a.y ^ b.y);
}
__device__ __forceinline__ uint32_t ham(const uint4& a, const uint4& b) {
    return __popc(a.x ^ b.x) + __popc(a.y ^ b.y) + __popc(a.z ^ b.z) + __popc(a.w ^ b.w);
}
// number of differing bytes (disidx_fields, flat_index.hpp:30-37, dbits = 8)
__device__ __forceinline__ uint32_t nz_bytes(uint32_t x) {
    x |= x >> 4;
    x |= x >> 2;
    x |= x >> 1;
    return __popc(x & 0x01010101u);
}
__device__ __forceinline__ uint32_t disidx(const uint2& a, const uint2& b) {
    return nz_bytes(a.x ^ b.x) + nz_bytes(a.y ^ b.y);
}
__device__ __forceinline__ uint32_t disidx(const uint4& a, const uint4& b) {
    return nz_bytes(a.x ^ b.x) + nz_bytes(a.y ^ b.y) + nz_bytes(a.z ^ b.z) + nz_bytes(a.w ^ b.w);
}
__device__ __forceinline__ uint32_t word(const uint2& c, int w) { return w == 0 ? c.x : c.y; }
__device__ __forceinline__ uint32_t word(const uint4& c, int w) {
    return w == 0 ? c.x : (w == 1 ? c.y : (w == 2 ? c.z : c.w));
}

// ADC through the stored-field LUT of one query (M rows of 256 floats), in sq order.
template <int M, class C>
__device__ __forceinline__ float adc(const float* __restrict__ L, const C& c) {
    float acc = L[word(c, 0) & 0xFFu];  // 0.0f + x == x for x >= +0
#pragma unroll
    for (int sq = 1; sq < M; ++sq) {
        const uint32_t f = (word(c, sq >> 2) >> (8 * (sq & 3))) & 0xFFu;
        acc = __fadd_rn(acc, L[sq * KSUB + f]);
    }
    return acc;
}

__device__ __forceinline__ uint32_t key_low(const ScanArgs& a, uint32_t pos) {
    return a.id_mode == ID_ARITH ? a.id0 + pos : __ldg(a.id32 + pos);
}

// Append a candidate key for batch query qg; track block completion.
__device__ __forceinline__ void append_candidate(const ScanArgs& a, uint32_t qg, unsigned long long key, uint32_t bs,
                                                 uint32_t* nreq_s, uint32_t* req_s) {
    const uint32_t slot = atomicAdd(&a.ccount[qg], 1u);
    if (slot >= a.cap) {
        atomicOr(a.overflow, 1u);
        return;
    }
    a.cand[(size_t)qg * a.cap + slot] = key;
    __threadfence();
    const uint32_t nblk = a.cap / bs;
    const uint32_t blk = slot / bs;
    if (atomicAdd(&a.bdone[(size_t)qg * nblk + blk], 1u) == bs - 1) {
        const uint32_t r = atomicAdd(nreq_s, 1u);
        if (r < MAXREQ) req_s[r] = (qg << 16) | blk;
    }
}

// k-th smallest (1-based) of n distinct keys in global memory; CTA-cooperative
// 8-pass radix select, keys streamed from L2 each pass.
template <int NT>
__device__ unsigned long long block_select_kth(const unsigned long long* src, uint32_t n, uint32_t kk,
                                               uint32_t* hist, unsigned long long* prefix_s, uint32_t* k_s) {
    unsigned long long prefix = 0, mask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += NT) {
            const unsigned long long v = __ldcg(src + i);
            if ((v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 0xFFu], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            uint32_t c[8], s = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) { c[j] = hist[lane * 8 + j]; s += c[j]; }
            uint32_t incl = s;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += o;
            }
            const uint32_t excl = incl - s;
            if (excl < kk && kk <= incl) {
                uint32_t r = kk - excl;
                int digit = lane * 8 + 7;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (r <= c[j]) { digit = lane * 8 + j; break; }
                    r -= c[j];
                }
                *prefix_s = prefix | ((unsigned long long)digit << shift);
                *k_s = r;
            }
        }
        __syncthreads();
        prefix = *prefix_s;
        kk = *k_s;
        mask |= 0xFFull << shift;
    }
    return prefix;
}

template <int M, int Q, int W, int STRAT>
__global__ void __launch_bounds__(W * 32, 1) scan_kernel(const ScanArgs a, uint32_t bs) {
    using C = typename CodeT<M>::T;
    constexpr int NT = W * 32;
    constexpr int TC = 16384 / M;   // codes per 16 KB tile
    constexpr int CPW = TC / W;     // codes per warp per tile
    constexpr bool USE_LUT = (STRAT == DUAL || STRAT == ADC);
    constexpr int LUT_FLOATS = USE_LUT ? Q * M * KSUB : 0;

    extern __shared__ __align__(128) uint8_t smem[];
    float* lut = reinterpret_cast<float*>(smem);
    C* tiles = reinterpret_cast<C*>(smem + LUT_FLOATS * 4);
    C* qu_code = tiles + STAGES * TC;                          // W x QCAP
    uint2* qu_meta = reinterpret_cast<uint2*>(qu_code + W * QCAP);  // (pos, q)

    __shared__ __align__(8) uint64_t full_bar[STAGES];
    __shared__ unsigned long long thr_s[Q];
    __shared__ C qc_s[Q];
    __shared__ uint32_t unit_s, nreq_s, group_s;
    __shared__ uint32_t req_s[MAXREQ];
    __shared__ uint32_t sel_hist[256];
    __shared__ unsigned long long sel_prefix_s;
    __shared__ uint32_t sel_k_s;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full_bar[s], 1);
        fence_mbar_init();
        nreq_s = 0;
        group_s = 0xFFFFFFFFu;
    }
    __syncthreads();

    C* myq_code = qu_code + warp * QCAP;
    uint2* myq_meta = qu_meta + warp * QCAP;
    uint32_t seq = 0;  // tiles consumed by this CTA (stage = seq % STAGES, parity = (seq / STAGES) & 1)

    for (;;) {
        if (threadIdx.x == 0) unit_s = atomicAdd(a.work, 1u);
        __syncthreads();
        const uint32_t unit = unit_s;
        if (unit >= a.units) break;
        const uint32_t g = unit % a.ngroups, chunk = unit / a.ngroups;
        const uint32_t q0 = g * Q;
        const uint32_t nqh = min((uint32_t)Q, a.nqb - q0);
        const uint64_t t0 = (uint64_t)chunk * a.tiles_per_chunk;
        const uint32_t ntile = (uint32_t)min((uint64_t)a.tiles_per_chunk, a.ntiles - t0);

        // producer prologue: fill the ring
        auto issue = [&](uint32_t s_seq, uint64_t t) {
            const uint32_t s = s_seq % STAGES;
            const uint64_t first = t * a.tile_stride * TC;
            const uint64_t cnt = min((uint64_t)TC, a.n - first);
            const uint32_t bytes = (uint32_t)((cnt * M + 15) & ~15ull);
            mbar_arrive_expect_tx(&full_bar[s], bytes);
            bulk_g2s(tiles + s * TC, a.codes + first * M, bytes, &full_bar[s]);
        };
        if (threadIdx.x == 0) {
            for (uint32_t j = 0; j < min((uint32_t)STAGES, ntile); ++j) issue(seq + j, t0 + j);
        }
        // per-group state: LUTs (only when the group changes), query codes, thresholds
        if (group_s != g) {
            if (USE_LUT) {
                const float4* src = reinterpret_cast<const float4*>(a.lutp + (size_t)q0 * M * KSUB);
                float4* dst = reinterpret_cast<float4*>(lut);
                const uint32_t n4 = nqh * M * KSUB / 4;
                for (uint32_t i = threadIdx.x; i < n4; i += NT) dst[i] = __ldg(src + i);
            }
            if (threadIdx.x < Q)
                qc_s[threadIdx.x] = threadIdx.x < nqh ? reinterpret_cast<const C*>(a.qcodes)[q0 + threadIdx.x] : C{};
        }
        if (threadIdx.x < Q) thr_s[threadIdx.x] = threadIdx.x < nqh ? __ldcg(a.thr + q0 + threadIdx.x) : 0ull;
        __syncthreads();
        if (threadIdx.x == 0) group_s = g;

        C qc[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) qc[q] = qc_s[q];
        uint32_t surv[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) surv[q] = 0;
        uint32_t qn = 0;  // entries in this warp's queue

        // drain `cnt` queued survivors (lanes < cnt busy): ADC + candidate test
        auto drain = [&](uint32_t cnt) {
            __syncwarp();
            if ((uint32_t)lane < cnt) {
                const C code = myq_code[lane];
                const uint2 meta = myq_meta[lane];
                const float* L = lut + meta.y * (M * KSUB);
                const float score = adc<M>(L, code);
                const uint32_t sb = __float_as_uint(score);
                const unsigned long long thr = thr_s[meta.y];
                if (sb <= (uint32_t)(thr >> 32)) {
                    const unsigned long long key = ((unsigned long long)sb << 32) | key_low(a, meta.x);
                    if (key < thr) append_candidate(a, q0 + meta.y, key, bs, &nreq_s, req_s);
                }
            }
            __syncwarp();
        };

        for (uint32_t j = 0; j < ntile; ++j) {
            const uint32_t s = (seq + j) % STAGES;
            mbar_wait(&full_bar[s], ((seq + j) / STAGES) & 1u);
            const C* T = tiles + s * TC;
            const uint64_t tfirst = (t0 + j) * a.tile_stride * TC;
            const uint32_t tcnt = (uint32_t)min((uint64_t)TC, a.n - tfirst);
#pragma unroll 1
            for (int i = 0; i < CPW / 32; ++i) {
                const uint32_t li = warp * CPW + i * 32 + lane;
                const bool in = li < tcnt;
                const C code = T[li];
                const uint32_t pos = (uint32_t)(tfirst + li);
                if constexpr (STRAT == DUAL) {
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        if (q >= (int)nqh) break;
                        const bool pass = in && ham(code, qc[q]) <= a.tau;
                        const uint32_t b = __ballot_sync(0xffffffffu, pass);
                        if (b) {
                            const uint32_t nb = __popc(b);
                            surv[q] += nb;
                            if (pass) {
                                const uint32_t at = qn + __popc(b & lanemask_lt());
                                myq_code[at] = code;
                                myq_meta[at] = make_uint2(pos, (uint32_t)q);
                            }
                            qn += nb;
                            if (qn >= 32) {
                                drain(32);
                                qn -= 32;
                                if ((uint32_t)lane < qn) {
                                    myq_code[lane] = myq_code[32 + lane];
                                    myq_meta[lane] = myq_meta[32 + lane];
                                }
                                __syncwarp();
                            }
                        }
                    }
                } else {
                    // adc / binary / disidx: every code is scored for every query
#pragma unroll 1
                    for (int q = 0; q < (int)nqh; ++q) {
                        float score;
                        if constexpr (STRAT == ADC) score = adc<M>(lut + q * (M * KSUB), code);
                        else if constexpr (STRAT == BINARY) score = (float)ham(code, qc_s[q]);
                        else score = (float)disidx(code, qc_s[q]);
                        if (in) {
                            const uint32_t sb = __float_as_uint(score);
                            const unsigned long long thr = thr_s[q];
                            if (sb <= (uint32_t)(thr >> 32)) {
                                const unsigned long long key = ((unsigned long long)sb << 32) | key_low(a, pos);
                                if (key < thr) append_candidate(a, q0 + q, key, bs, &nreq_s, req_s);
                            }
                        }
                    }
                }
            }
            __syncthreads();  // stage s fully consumed (queued survivors hold copies of their codes)
            if (threadIdx.x == 0 && j + STAGES < ntile) issue(seq + j + STAGES, t0 + j + STAGES);
            // threshold maintenance: selects requested by appends of this CTA
            const uint32_t nr = min(nreq_s, (uint32_t)MAXREQ);
            for (uint32_t r = 0; r < nr; ++r) {
                const uint32_t qg = req_s[r] >> 16, blk = req_s[r] & 0xFFFFu;
                __threadfence();
                const unsigned long long kth = block_select_kth<NT>(a.cand + (size_t)qg * a.cap + (size_t)blk * bs,
                                                                    bs, a.k, sel_hist, &sel_prefix_s, &sel_k_s);
                if (threadIdx.x == 0) atomicMin(a.thr + qg, kth);
            }
            __syncthreads();
            if (threadIdx.x == 0) nreq_s = 0;
            if (threadIdx.x < nqh) thr_s[threadIdx.x] = __ldcg(a.thr + q0 + threadIdx.x);
            __syncthreads();
        }
        seq += ntile;
        if constexpr (STRAT == DUAL) {
            if (qn) drain(qn);
            if (lane == 0)
                for (int q = 0; q < Q; ++q)
                    if (q < (int)nqh && surv[q]) atomicAdd(a.surv + q0 + q, (unsigned long long)surv[q]);
        }
        __syncthreads();
    }
}

template <int M, int Q, int W, int STRAT>
static void launch_one(const ScanArgs& a, int num_sms, cudaStream_t s) {
    constexpr int TC = 16384 / M;
    constexpr bool USE_LUT = (STRAT == DUAL || STRAT == ADC);
    const size_t smem = (USE_LUT ? (size_t)Q * M * KSUB * 4 : 0) + (size_t)STAGES * TC * M +
                        (size_t)W * QCAP * (M + 8);
    auto kfn = scan_kernel<M, Q, W, STRAT>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const uint32_t bs = a.k * 4 > (uint32_t)BS ? a.k * 4 : (uint32_t)BS;
    const unsigned grid = (unsigned)((uint64_t)num_sms < (uint64_t)a.units ? (uint64_t)num_sms : (uint64_t)a.units);
    kfn<<<grid, W * 32, smem, s>>>(a, bs);
    count_launch();
}

int scan_queries_per_cta(uint32_t m) { return m == 8 ? 16 : 8; }

void launch_scan(const ScanArgs& a, int strategy, uint32_t m, int num_sms, cudaStream_t s) {
    // Q queries per CTA: Q x m x 1 KB of LUTs must fit next to the tile ring.
    if (m == 8) {
        switch (strategy) {
            case DUAL: launch_one<8, 16, 16, DUAL>(a, num_sms, s); break;
            case ADC: launch_one<8, 16, 16, ADC>(a, num_sms, s); break;
            case BINARY: launch_one<8, 16, 16, BINARY>(a, num_sms, s); break;
            default: launch_one<8, 16, 16, DISIDX>(a, num_sms, s); break;
        }
    } else {
        switch (strategy) {
            case DUAL: launch_one<16, 8, 16, DUAL>(a, num_sms, s); break;
            case ADC: launch_one<16, 8, 16, ADC>(a, num_sms, s); break;
            case BINARY: launch_one<16, 8, 16, BINARY>(a, num_sms, s); break;
            default: launch_one<16, 8, 16, DISIDX>(a, num_sms, s); break;
        }
    }
}

}  // namespace pb
