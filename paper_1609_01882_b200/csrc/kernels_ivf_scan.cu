// kernels_ivf_scan.cu -- K6: the IVF inverted-list scan (configs 2/4; search_coarse
// SPEC.md:382-390).
//
// A work unit is (query, probe, r0, r1): rows [r0, r1) of the probed cell's list,
// from the probe-count kernel (kernels_ivf.cu).  One CTA per unit (dynamic), K6W
// warps.  Thread 0 pulls the item's residual LUT (K1r output, 8 / 16 KB) into
// shared memory with a 1-D bulk copy (TMA, mbarrier completion) while every lane
// loads the item's query code and bound into registers, so a unit costs one CTA
// barrier.  Each warp streams 4 codes per lane (ld.global.cs: no reuse across
// units), tests them -- Hamming filter (hamming_bytes flat_index.hpp:14-27, kept
// iff h <= tau) -- and compacts the survivors by ballot into a
// per-warp queue of (code, row) entries in shared memory; every 32 entries are
// drained with all lanes busy:
// ADC (adc_distance pq.cpp:121-128: __fadd_rn in sub-quantizer order, exact
// half-sum early exit, code_ops.cuh) and the candidate test against the query's
// bound.  Shared memory is addressed through 32-bit window addresses held in
// registers (no generic-pointer rebuilds in the loop).
#include "code_ops.cuh"

namespace pb {

#ifndef POLY_K6_WARPS
#define POLY_K6_WARPS 4
#endif
#ifndef POLY_K6_PREFETCH  // 1: software-pipelined code loads (one block ahead)
#define POLY_K6_PREFETCH 1
#endif
#ifndef POLY_K6_MINB
#define POLY_K6_MINB 10  // CTAs per SM the register budget is sized for (m = 8; A/B with the prefetch: 10 > 12, 8)
#endif
constexpr int K6W = POLY_K6_WARPS;
constexpr uint32_t K6_QN = 64;  // queue entries per warp: < 32 carried + one ballot step

__device__ __forceinline__ void s_st128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint4 s_ld128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
                 : "memory");
    return v;
}
__device__ __forceinline__ void s_st32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t s_ld32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ float s_ldf(uint32_t a) {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}
__device__ __forceinline__ uint2 ld_stream(const uint2* p) { return __ldcs(p); }
__device__ __forceinline__ uint4 ld_stream(const uint4* p) { return __ldcs(p); }

// LUT entry address of stored field byte `sq` of the code: L + sq KB + 4 * field
template <class C>
__device__ __forceinline__ uint32_t lut_at(uint32_t L, const C& c, int sq) {
    const uint32_t f = __byte_perm(word(c, sq >> 2), 0u, 0x4440u + (uint32_t)(sq & 3));
    return L + (uint32_t)(sq * KSUB * 4) + (f << 2);
}

// adc_distance with the exact half-sum exit (code_ops.cuh adc_bounded), LUT at shared address L
template <int M, class C>
__device__ __forceinline__ float adc_sh(uint32_t L, const C& c, uint32_t bound_bits) {
    float acc = s_ldf(lut_at(L, c, 0));
#pragma unroll
    for (int sq = 1; sq < M / 2; ++sq) acc = __fadd_rn(acc, s_ldf(lut_at(L, c, sq)));
    if (__float_as_uint(acc) > bound_bits) return __int_as_float(0x7f800000);
#pragma unroll
    for (int sq = M / 2; sq < M; ++sq) acc = __fadd_rn(acc, s_ldf(lut_at(L, c, sq)));
    return acc;
}

template <int M>
struct K6Smem {
    static constexpr uint32_t LUT_BYTES = (uint32_t)(M * KSUB * 4);
    // queue entry: m = 8 one 16-byte {code.x, code.y, row, 0}; m = 16 a 16-byte code + a 4-byte row
    static constexpr uint32_t QW = K6_QN * (M == 8 ? 16u : 20u);
    static constexpr uint32_t TOTAL = LUT_BYTES + K6W * QW;
};

template <int M, int STRAT, bool PERQ>
__global__ void __launch_bounds__(K6W * 32, M == 8 ? POLY_K6_MINB : 8) ivf_list_scan_kernel(const IvfScanArgs a) {
    using C = typename CodeT<M>::T;
    using S = K6Smem<M>;
    extern __shared__ __align__(128) uint8_t k6s[];
    __shared__ __align__(8) uint64_t lut_bar;
    __shared__ uint32_t unit_s;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // shared-window addresses, made opaque so ptxas keeps them in registers instead of
    // rebuilding them from SR_CgaCtaId inside the loop
    const uint32_t lut0 = opaque_u32(smem_u32(k6s));
    const uint32_t qb = opaque_u32(lut0 + S::LUT_BYTES + warp * S::QW);  // this warp's queue
    const uint32_t qm = qb + K6_QN * 16u;                                // m = 16: row words
    const uint32_t lt = (1u << lane) - 1u, tau = a.tau;
    if (threadIdx.x == 0) {
        mbar_init(&lut_bar, 1);
        fence_mbar_init();
    }
    const uint32_t nunits = min(*a.nitems, a.items_cap);
    uint32_t phase = 0, surv_total = 0;
    for (;;) {
        __syncthreads();  // the previous unit's LUT and queues are no longer read
        if (threadIdx.x == 0) unit_s = atomicAdd(a.work, 1u);
        __syncthreads();
        const uint32_t u = unit_s;
        if (u >= nunits) break;
        const uint4 un = __ldg(a.items + u);  // (query, probe, r0, r1)
        const uint32_t qi = un.x, item = un.x * a.nprobe + un.y;
        if (threadIdx.x == 0) {  // the LUT by bulk copy; the barrier above ordered the prior generic reads
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&lut_bar, (uint32_t)(M * KSUB * 4));
            bulk_g2s(k6s, a.lutp + (size_t)item * M * KSUB, M * KSUB * 4, &lut_bar);
        }
        const uint32_t cell = (uint32_t)__ldg(a.probe_keys + item);
        const C qc = reinterpret_cast<const C*>(a.qcodes)[item];
        const unsigned long long thr = __ldcg(a.thr + qi);
        const uint64_t beg = __ldg(a.off + cell) + un.z;
        const uint32_t n = un.w - un.z, pos0 = (uint32_t)beg;
        const C* ci = reinterpret_cast<const C*>(a.codes) + beg;
        mbar_wait(&lut_bar, phase);
        phase ^= 1u;

        uint32_t qn = 0;
        // drain cnt entries from the queue head (lanes < cnt busy)
        auto drain = [&](uint32_t cnt) {
            __syncwarp();
            if (lane < cnt) {
                C cc;
                uint32_t row;
                if constexpr (M == 8) {
                    const uint4 e = s_ld128(qb + 16u * lane);
                    cc.x = e.x;
                    cc.y = e.y;
                    row = e.z;
                } else {
                    cc = s_ld128(qb + 16u * lane);
                    row = s_ld32(qm + 4u * lane);
                }
                float score;
                if constexpr (STRAT == DUAL || STRAT == ADC) score = adc_sh<M>(lut0, cc, (uint32_t)(thr >> 32));
                else if constexpr (STRAT == BINARY) score = (float)ham(cc, qc);
                else score = (float)disidx(cc, qc);
                const uint32_t sb = __float_as_uint(score);
                if (sb <= (uint32_t)(thr >> 32)) {
                    const unsigned long long key = ((unsigned long long)sb << 32) | __ldg(a.low + pos0 + row);
                    if (key < thr) {
                        const uint32_t slot = atomicAdd(&a.ccount[qi], 1u);
                        if (slot < a.cap) a.cand[(size_t)qi * a.cap + slot] = key;
                        else a.ovq[qi] = 1u;  // list full: the rescue scan re-ranks this query exactly
                    }
                }
            }
            __syncwarp();
        };
#if POLY_K6_PREFETCH
        // the next block's codes are loaded before this block is filtered and drained
        C cn[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint32_t row = warp * 128u + 32u * v + lane;
            if (row < n) cn[v] = ld_stream(ci + row);
        }
#endif
        for (uint32_t rb = warp * 128u; rb < n; rb += 128u * K6W) {
            C c[4];
#if POLY_K6_PREFETCH
#pragma unroll
            for (int v = 0; v < 4; ++v) c[v] = cn[v];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint32_t row = rb + 128u * K6W + 32u * v + lane;
                if (row < n) cn[v] = ld_stream(ci + row);
            }
#else
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint32_t row = rb + 32u * v + lane;
                if (row < n) c[v] = ld_stream(ci + row);
            }
#endif
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint32_t row = rb + 32u * v + lane;
                bool pass = row < n;
                if constexpr (STRAT == DUAL) pass = pass && ham(c[v], qc) <= tau;
                if constexpr (PERQ && (STRAT == DUAL || STRAT == ADC)) {  // stats mode: per-query count + id hash
                    if (pass) {
                        atomicAdd(a.surv_q + qi, 1ull);
                        atomicAdd(a.hash_q + qi, (unsigned long long)mix64(__ldg(a.low + pos0 + row)));
                    }
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, pass);
                if (!bal) continue;
                if (pass) {
                    const uint32_t at = qn + __popc(bal & lt);
                    if constexpr (M == 8) {
                        s_st128(qb + 16u * at, c[v].x, c[v].y, row, 0u);
                    } else {
                        s_st128(qb + 16u * at, c[v].x, c[v].y, c[v].z, c[v].w);
                        s_st32(qm + 4u * at, row);
                    }
                }
                const uint32_t nb = __popc(bal);
                qn += nb;
                surv_total += nb;
                if (qn >= 32) {
                    drain(32);
                    qn -= 32;
                    if (lane < qn) {  // carry the rest to the queue head
                        const uint4 e = s_ld128(qb + 16u * (32u + lane));
                        s_st128(qb + 16u * lane, e.x, e.y, e.z, e.w);
                        if constexpr (M == 16) s_st32(qm + 4u * lane, s_ld32(qm + 4u * (32u + lane)));
                    }
                    __syncwarp();
                }
            }
        }
        if (qn) drain(qn);
    }
    if (STRAT == DUAL && lane == 0 && surv_total) atomicAdd(a.surv_total, (unsigned long long)surv_total);
}

template <int M, int STRAT>
static void launch_list_one(const IvfScanArgs& a, int num_sms, cudaStream_t s) {
    using S = K6Smem<M>;
    const bool perq = a.surv_q != nullptr;
    auto kfn = perq ? ivf_list_scan_kernel<M, STRAT, true> : ivf_list_scan_kernel<M, STRAT, false>;
    set_max_smem((const void*)kfn, S::TOTAL);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, K6W * 32, S::TOTAL) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    kfn<<<(unsigned)(num_sms * per_sm), K6W * 32, S::TOTAL, s>>>(a);
    count_launch();
}

template <int M>
static void launch_list_m(const IvfScanArgs& a, int strategy, int num_sms, cudaStream_t s) {
    switch (strategy) {
        case DUAL: launch_list_one<M, DUAL>(a, num_sms, s); break;
        case ADC: launch_list_one<M, ADC>(a, num_sms, s); break;
        case BINARY: launch_list_one<M, BINARY>(a, num_sms, s); break;
        default: launch_list_one<M, DISIDX>(a, num_sms, s); break;
    }
}

void launch_ivf_scan(const IvfScanArgs& a, int strategy, uint32_t m, int num_sms, cudaStream_t s) {
    if (a.nq == 0) return;
    if (m == 8) launch_list_m<8>(a, strategy, num_sms, s);
    else launch_list_m<16>(a, strategy, num_sms, s);
}

}  // namespace pb
