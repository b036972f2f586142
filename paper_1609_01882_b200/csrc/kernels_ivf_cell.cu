// kernels_ivf_cell.cu -- K6g: the IVF list scan in cell-major order (configs 2/4).
//
// search_coarse visits, for every query, the lists of its
// nprobe nearest cells.  K6 (kernels_ivf.cu) walks those (query, probe) items
// one at a time, so a list probed by B queries of the batch is streamed from
// HBM B times.  K6g groups the batch's items by cell instead:
//
//   cw_count    per query, per probe of the round: ccnt[cell] += 1
//   cw_plan     one CTA: exclusive scans of the per-cell item counts and of the
//               per-cell unit counts; a unit is (cell, group of <= G items,
//               rows [r0, r1) of the cell's list)
//   cw_scatter  per query, per probe: the item index q * nprobe + p goes to its
//               cell's slot range (order within a cell is irrelevant: results
//               order by (score, id), never by visit order)
//   K6g         one CTA per unit (dynamic): the group's G residual LUTs (K1r
//               output) sit in shared memory, each warp loads 4 codes per lane
//               once and tests them against every query of the group --
//               Hamming filter (hamming_bytes flat_index.hpp:14-27, h <= tau,
//               SPEC.md:310), survivors compacted by ballot into a per-warp
//               queue, drained 32 at a time with the ADC sum (adc_distance
//               pq.cpp:121-128, __fadd_rn in sub-quantizer order, exact early
//               exit) and the candidate test against the query's bound.
//
// The per-pair arithmetic is K6's (code_ops.cuh), so results are identical;
// only the visit order and the code reuse change.  Codes are read from HBM
// once per unit, i.e. once per group of G queries probing the cell.
#include "code_ops.cuh"

namespace pb {

// ------------------------------------------------------------------ plan
// round r of query q visits probes [lo, hi): r = 0 -> [0, min(split, ne)), r = 1 -> [min(split, ne), ne)
__device__ __forceinline__ void cw_range(const CellWork& w, uint32_t q, uint32_t& lo, uint32_t& hi) {
    const uint32_t ne = w.np_eff[q];
    const uint32_t sp = w.split ? min(w.split[q], ne) : 0u;
    lo = w.round ? sp : 0u;
    hi = w.round ? ne : (w.split ? sp : ne);
}

__global__ void cw_count_kernel(const CellWork w) {
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (q >= w.nq) return;
    uint32_t lo, hi;
    cw_range(w, q, lo, hi);
    for (uint32_t p = lo + lane; p < hi; p += 32) atomicAdd(&w.ccnt[(uint32_t)w.probe_keys[(size_t)q * w.nprobe + p]], 1u);
}

__global__ void cw_scatter_kernel(const CellWork w) {
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (q >= w.nq) return;
    uint32_t lo, hi;
    cw_range(w, q, lo, hi);
    for (uint32_t p = lo + lane; p < hi; p += 32) {
        const uint32_t item = q * w.nprobe + p;
        const uint32_t slot = atomicAdd(&w.ccnt[(uint32_t)w.probe_keys[item]], 1u);  // ccnt = cursors after the plan
        w.sorted[slot] = item;
    }
}

// One CTA of CW_PLAN_T threads over all cells: cell c's items go to slots
// [cio(c), cio(c) + cnt(c)); its units are (cell | n_g << 24, first slot of the
// group, r0, r1), rows split at w.rows, groups of <= w.g items.  ccnt[c] is
// overwritten with cio(c) (the scatter's cursor).
constexpr uint32_t CW_PLAN_T = 1024;

__device__ __forceinline__ uint32_t cw_units_of(uint32_t cnt, uint64_t len, uint32_t g, uint32_t rows) {
    if (!cnt || !len) return 0u;
    return ((cnt + g - 1) / g) * (uint32_t)((len + rows - 1) / rows);
}

template <typename T>
__device__ __forceinline__ T cw_block_excl(T v, T* sh, T& total) {  // exclusive block scan (CW_PLAN_T threads)
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += x;
    }
    if (lane == 31) sh[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T s = lane < CW_PLAN_T / 32 ? sh[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T x = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= (uint32_t)o) s += x;
        }
        sh[lane] = s;  // inclusive per warp
    }
    __syncthreads();
    const T before = warp ? sh[warp - 1] : T(0);
    total = sh[CW_PLAN_T / 32 - 1];
    __syncthreads();
    return before + incl - v;
}

__global__ void __launch_bounds__(CW_PLAN_T) cw_plan_kernel(const CellWork w, const uint64_t* __restrict__ off,
                                                            uint32_t nlist) {
    __shared__ uint32_t sh_i[32];
    __shared__ unsigned long long sh_u[32];
    const uint32_t per = (nlist + CW_PLAN_T - 1) / CW_PLAN_T;
    const uint32_t c0 = min(nlist, threadIdx.x * per), c1 = min(nlist, c0 + per);
    uint32_t si = 0;
    unsigned long long su = 0;
    for (uint32_t c = c0; c < c1; ++c) {
        const uint32_t cnt = w.ccnt[c];
        si += cnt;
        su += cw_units_of(cnt, off[c + 1] - off[c], w.g, w.rows);
    }
    uint32_t ti;
    unsigned long long tu;
    uint32_t io = cw_block_excl<uint32_t>(si, sh_i, ti);
    unsigned long long uo = cw_block_excl<unsigned long long>(su, sh_u, tu);
    if (threadIdx.x == 0) {
        *w.nunits = tu < 0xFFFFFFFFull ? (uint32_t)tu : 0xFFFFFFFFu;
        if (tu > w.units_cap) atomicOr(w.overflow, 1u);
    }
    for (uint32_t c = c0; c < c1; ++c) {
        const uint32_t cnt = w.ccnt[c];
        const uint64_t b = off[c], len = off[c + 1] - b;
        w.ccnt[c] = io;
        if (cnt && len) {
            const uint32_t ng = (cnt + w.g - 1) / w.g;
            const uint32_t nr = (uint32_t)((len + w.rows - 1) / w.rows);
            for (uint32_t ri = 0; ri < nr; ++ri)
                for (uint32_t gi = 0; gi < ng; ++gi) {
                    if (uo < w.units_cap) {
                        const uint32_t gn = min(w.g, cnt - gi * w.g);
                        const uint32_t r0 = ri * w.rows;
                        const uint64_t e1 = (uint64_t)(ri + 1) * w.rows;
                        const uint32_t r1 = (uint32_t)(len < e1 ? len : e1);
                        w.units[uo] = make_uint4(c | (gn << 24), io + gi * w.g, r0, r1);
                    }
                    ++uo;
                }
        }
        io += cnt;
    }
}

void launch_cell_plan(const CellWork& w, const uint64_t* off, uint32_t nlist, cudaStream_t s) {
    if (w.nq == 0) return;  // (ccnt zeroed by the caller)
    const unsigned grid = (w.nq * 32 + 255) / 256;
    cw_count_kernel<<<grid, 256, 0, s>>>(w);
    count_launch();
    cw_plan_kernel<<<1, CW_PLAN_T, 0, s>>>(w, off, nlist);
    count_launch();
    cw_scatter_kernel<<<grid, 256, 0, s>>>(w);
    count_launch();
}

// ------------------------------------------------------------------ K6g
#ifndef POLY_K6G_WARPS
#define POLY_K6G_WARPS 8
#endif
constexpr int K6G_WARPS = POLY_K6G_WARPS;

__device__ __forceinline__ void g_sts(uint32_t a, const uint2& c) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(c.x), "r"(c.y) : "memory");
}
__device__ __forceinline__ void g_sts(uint32_t a, const uint4& c) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(c.x), "r"(c.y), "r"(c.z), "r"(c.w) : "memory");
}
__device__ __forceinline__ void g_sts(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void g_lds(uint32_t a, uint2& c) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(c.x), "=r"(c.y) : "r"(a) : "memory");
}
__device__ __forceinline__ void g_lds(uint32_t a, uint4& c) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "r"(a) : "memory");
}
__device__ __forceinline__ void g_lds(uint32_t a, uint32_t& v) {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
}
__device__ __forceinline__ float g_ldsf(uint32_t a) {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}

// ADC through the LUT at shared address L (bytes), with the exact half-sum exit (code_ops.cuh adc_bounded)
template <int M, class C>
__device__ __forceinline__ float g_adc_bounded(uint32_t L, const C& c, uint32_t bound_bits) {
    float acc = g_ldsf(L + 4u * field(c, 0));
#pragma unroll
    for (int sq = 1; sq < M / 2; ++sq) acc = __fadd_rn(acc, g_ldsf(L + 4u * (sq * KSUB + field(c, sq))));
    if (__float_as_uint(acc) > bound_bits) return __int_as_float(0x7f800000);
#pragma unroll
    for (int sq = M / 2; sq < M; ++sq) acc = __fadd_rn(acc, g_ldsf(L + 4u * (sq * KSUB + field(c, sq))));
    return acc;
}

template <int M, int G>
struct K6gSmem {
    static constexpr int LS = M * KSUB + 4;  // floats per LUT (+4: groups' same fields on different banks)
    static constexpr int QN = 64;            // per-warp queue entries
    static constexpr size_t LUT_BYTES = (size_t)G * LS * 4;
    static constexpr size_t Q_BYTES = (size_t)K6G_WARPS * QN * (sizeof(typename CodeT<M>::T) + 4);
    static constexpr size_t TOTAL = LUT_BYTES + Q_BYTES;
};

template <int M, int G, int STRAT, bool PERQ>
__global__ void __launch_bounds__(K6G_WARPS * 32) ivf_cell_scan_kernel(const IvfScanArgs a, const CellWork w) {
    using C = typename CodeT<M>::T;
    using SMEM = K6gSmem<M, G>;
    constexpr int NT = K6G_WARPS * 32;
    extern __shared__ __align__(16) uint8_t g_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lut_base = smem_u32(g_smem);
    const uint32_t qcs = lut_base + (uint32_t)SMEM::LUT_BYTES + warp * SMEM::QN * (uint32_t)(sizeof(C) + 4);
    const uint32_t qps = qcs + SMEM::QN * (uint32_t)sizeof(C);
    const uint32_t lt = (1u << lane) - 1u, tau = a.tau;
    const uint32_t nunits = min(*w.nunits, w.units_cap);
    __shared__ C qc_s[G];
    __shared__ unsigned long long thr_s[G];
    __shared__ uint32_t qi_s[G];
    __shared__ uint32_t unit_s;
    uint32_t surv_total = 0;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) unit_s = atomicAdd(w.work, 1u);
        __syncthreads();
        const uint32_t u = unit_s;
        if (u >= nunits) break;
        const uint4 un = w.units[u];
        const uint32_t cell = un.x & 0xFFFFFFu, ng = un.x >> 24;
        // stage the group's LUTs (float4), query codes and bounds
        {
            constexpr uint32_t PER = M * KSUB / 4;
            for (uint32_t i = threadIdx.x; i < ng * PER; i += NT) {
                const uint32_t g = i / PER, o = i % PER;
                const uint32_t item = w.sorted[un.y + g];
                const float4 v = __ldg(reinterpret_cast<const float4*>(a.lutp + (size_t)item * M * KSUB) + o);
                reinterpret_cast<float4*>(g_smem)[g * (SMEM::LS / 4) + o] = v;
            }
            if (threadIdx.x < ng) {
                const uint32_t item = w.sorted[un.y + threadIdx.x];
                const uint32_t qi = item / a.nprobe;
                qi_s[threadIdx.x] = qi;
                qc_s[threadIdx.x] = reinterpret_cast<const C*>(a.qcodes)[item];
                thr_s[threadIdx.x] = __ldcg(a.thr + qi);
            }
        }
        __syncthreads();
        const uint64_t beg = a.off[cell] + un.z;
        const uint32_t n = un.w - un.z, pos0 = (uint32_t)beg;
        const C* ci = reinterpret_cast<const C*>(a.codes) + beg;
        C qc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) qc[g] = qc_s[g < (int)ng ? g : 0];
        uint32_t qn = 0;
        // drain cnt queued entries: entry = (row << 4) | g
        auto drain = [&](uint32_t cnt) {
            __syncwarp();
            if ((uint32_t)lane < cnt) {
                C cc;
                uint32_t e;
                g_lds(qcs + lane * (uint32_t)sizeof(C), cc);
                g_lds(qps + 4u * lane, e);
                const uint32_t g = e & 15u, pos = pos0 + (e >> 4);
                const unsigned long long thr = thr_s[g];
                float score;
                if constexpr (STRAT == DUAL || STRAT == ADC)
                    score = g_adc_bounded<M>(lut_base + 4u * g * SMEM::LS, cc, (uint32_t)(thr >> 32));
                else if constexpr (STRAT == BINARY) score = (float)ham(cc, qc_s[g]);
                else score = (float)disidx(cc, qc_s[g]);
                const uint32_t sb = __float_as_uint(score);
                if (sb <= (uint32_t)(thr >> 32)) {
                    const unsigned long long key = ((unsigned long long)sb << 32) | __ldg(a.low + pos);
                    if (key < thr) {
                        const uint32_t qi = qi_s[g];
                        const uint32_t slot = atomicAdd(&a.ccount[qi], 1u);
                        if (slot < a.cap) a.cand[(size_t)qi * a.cap + slot] = key;
                        else a.ovq[qi] = 1u;  // list full: the rescue scan re-ranks this query exactly
                    }
                }
            }
            __syncwarp();
        };
        auto push = [&](bool pass, const C& c, uint32_t row, uint32_t g) {
            const uint32_t bal = __ballot_sync(0xffffffffu, pass);
            if (!bal) return;
            if (pass) {
                const uint32_t at = qn + __popc(bal & lt);
                g_sts(qcs + at * (uint32_t)sizeof(C), c);
                g_sts(qps + 4u * at, (row << 4) | g);
            }
            qn += __popc(bal);
            if (qn >= 32) {
                drain(32);
                qn -= 32;
                if ((uint32_t)lane < qn) {  // carry the overflow to the queue head
                    C cc;
                    uint32_t e;
                    g_lds(qcs + (32u + lane) * (uint32_t)sizeof(C), cc);
                    g_lds(qps + 4u * (32u + lane), e);
                    g_sts(qcs + lane * (uint32_t)sizeof(C), cc);
                    g_sts(qps + 4u * lane, e);
                }
                __syncwarp();
            }
        };
        for (uint32_t r0 = warp * 128; r0 < n; r0 += 128 * K6G_WARPS) {
            C c[4];
            bool in[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint32_t r = r0 + v * 32 + lane;
                in[v] = r < n;
                if (in[v]) c[v] = __ldcs(ci + r);  // streamed once per group: evict-first
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint32_t row = r0 + v * 32 + lane;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    if (g >= (int)ng) break;
                    bool pass = in[v];
                    if constexpr (STRAT == DUAL) pass = pass && ham(c[v], qc[g]) <= tau;
                    if constexpr (PERQ && (STRAT == DUAL || STRAT == ADC)) {  // stats mode: per-query count + id hash
                        if (pass) {
                            atomicAdd(a.surv_q + qi_s[g], 1ull);
                            atomicAdd(a.hash_q + qi_s[g], (unsigned long long)mix64(__ldg(a.low + pos0 + row)));
                        }
                    }
                    if constexpr (STRAT == DUAL) surv_total += pass;
                    push(pass, c[v], row, (uint32_t)g);
                }
            }
        }
        if (qn) drain(qn);
    }
    if (STRAT == DUAL) {
        surv_total = __reduce_add_sync(0xffffffffu, surv_total);
        if (lane == 0 && surv_total) atomicAdd(a.surv_total, (unsigned long long)surv_total);
    }
}

template <int M, int G, int STRAT>
static void launch_cell_one(const IvfScanArgs& a, const CellWork& w, int num_sms, cudaStream_t s) {
    using SMEM = K6gSmem<M, G>;
    const size_t smem = SMEM::TOTAL;
    const bool perq = a.surv_q != nullptr;
    auto kfn = perq ? ivf_cell_scan_kernel<M, G, STRAT, true> : ivf_cell_scan_kernel<M, G, STRAT, false>;
    set_max_smem((const void*)kfn, smem);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, K6G_WARPS * 32, smem) != cudaSuccess) per_sm = 1;
    const unsigned grid = (unsigned)num_sms * (unsigned)(per_sm > 0 ? per_sm : 1);
    kfn<<<grid, K6G_WARPS * 32, smem, s>>>(a, w);
    count_launch();
}

template <int M, int G>
static void launch_cell_g(const IvfScanArgs& a, const CellWork& w, int strategy, int num_sms, cudaStream_t s) {
    switch (strategy) {
        case DUAL: launch_cell_one<M, G, DUAL>(a, w, num_sms, s); break;
        case ADC: launch_cell_one<M, G, ADC>(a, w, num_sms, s); break;
        case BINARY: launch_cell_one<M, G, BINARY>(a, w, num_sms, s); break;
        default: launch_cell_one<M, G, DISIDX>(a, w, num_sms, s); break;
    }
}

uint32_t cell_scan_group(uint32_t m) { return m == 8 ? 8u : 4u; }

void launch_ivf_cell_scan(const IvfScanArgs& a, const CellWork& w, int strategy, uint32_t m, int num_sms,
                          cudaStream_t s) {
    if (a.nq == 0) return;
    if (m == 8) launch_cell_g<8, 8>(a, w, strategy, num_sms, s);
    else launch_cell_g<16, 4>(a, w, strategy, num_sms, s);
}

}  // namespace pb
