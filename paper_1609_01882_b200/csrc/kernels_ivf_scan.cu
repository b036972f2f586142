// kernels_ivf_scan.cu -- K6: the IVF inverted-list scan (configs 2/4; search_coarse
// SPEC.md:382-390).
//
// A work unit is (query, probe, r0, r1): rows [r0, r1) of the probed cell's list,
// from the probe-count kernel (kernels_ivf.cu).  One CTA per unit (dynamic), K6W
// warps.  Thread 0 pulls the item's residual LUT (K1r output, 8 / 16 KB) into
// shared memory with a 1-D bulk copy (TMA, mbarrier completion) while every lane
// loads the item's query code and bound into registers, so a unit costs one CTA
// barrier.  Each warp streams 4 codes per lane (ld.global.cs: no reuse across
// units; the next block's loads are issued before the current block is tested),
// tests them -- Hamming filter (hamming_bytes flat_index.hpp:14-27, kept iff
// h <= tau) -- and pushes the survivors by ballot into a per-warp ring
// of (code, row) entries in shared memory; whenever the ring holds 32 entries they
// are drained with all lanes busy:
// ADC (adc_distance pq.cpp:121-128: __fadd_rn in sub-quantizer order, exact
// half-sum early exit, code_ops.cuh) and the candidate test against the query's
// bound.  Shared memory is addressed through 32-bit window addresses held in
// registers (no generic-pointer rebuilds in the loop).  A warp's ring is two dense arrays
// (row words, codes): dense pushes have no bank conflicts, the drain reads the code and
// only a candidate reads its row word; the row ring is aligned to its own size so that a
// slot's address is one LOP3 ((x & mask) | base).
#include "code_ops.cuh"

namespace pb {

#ifndef POLY_K6_WARPS
#define POLY_K6_WARPS 4
#endif
#ifndef POLY_K6_MINB
#define POLY_K6_MINB 10  // CTAs per SM the register budget is sized for (m = 8; A/B: 10 > 12, 8)
#endif
constexpr int K6W = POLY_K6_WARPS;
constexpr uint32_t K6_QN = 128;            // ring entries per warp: < 32 carried + two ballot steps (power of two)
constexpr uint32_t K6_ROWRING = K6_QN * 4u;  // bytes of a warp's ring of row words = its alignment

__device__ __forceinline__ void s_st128_if(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w, bool p) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t@p st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"r"(a),
        "r"(x), "r"(y), "r"(z), "r"(w), "r"((uint32_t)p)
        : "memory");
}
__device__ __forceinline__ void s_st64_if(uint32_t a, uint32_t x, uint32_t y, bool p) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t@p st.shared.v2.u32 [%0], {%1, %2};\n\t}" ::"r"(a), "r"(x),
                 "r"(y), "r"((uint32_t)p)
                 : "memory");
}
__device__ __forceinline__ void s_st32_if(uint32_t a, uint32_t v, bool p) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u32 [%0], %1;\n\t}" ::"r"(a), "r"(v),
                 "r"((uint32_t)p)
                 : "memory");
}
__device__ __forceinline__ uint4 s_ld128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
                 : "memory");
    return v;
}
__device__ __forceinline__ uint2 s_ld64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
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
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {  // 16-byte aligned address and size
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
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
    // a warp's ring is two dense arrays (no bank conflicts on the pushes): K6_QN row words and
    // K6_QN codes; the row rings start at the next multiple of K6_ROWRING after the LUT (one of slack)
    static constexpr uint32_t TOTAL = LUT_BYTES + K6_ROWRING + K6W * K6_QN * (4u + (uint32_t)M);
};

template <int M, int STRAT, bool PERQ>
__global__ void __launch_bounds__(K6W * 32, M == 8 ? POLY_K6_MINB : 8) ivf_list_scan_kernel(const IvfScanArgs a) {
    using C = typename CodeT<M>::T;
    using S = K6Smem<M>;
    extern __shared__ __align__(128) uint8_t k6s[];
    __shared__ __align__(8) uint64_t lut_bar;
    __shared__ uint32_t unit_s[2];
    __shared__ uint4 item_s[2];
    const uint32_t lane = opaque_u32(threadIdx.x & 31), warp = threadIdx.x >> 5;
    // shared-window addresses, made opaque so ptxas keeps them in registers instead of
    // rebuilding them from SR_CgaCtaId inside the loop
    const uint32_t lut0 = opaque_u32(smem_u32(k6s));
    const uint32_t ring0 = (lut0 + S::LUT_BYTES + K6_ROWRING - 1u) & ~(K6_ROWRING - 1u);
    const uint32_t qr = opaque_u32(ring0 + warp * K6_ROWRING);  // this warp's ring of row words (aligned to its size)
    // its ring of codes at qc0: slot address = qc0 + (M / 4) * (row-word address - qr) = (M / 4) * address + qk
    const uint32_t qk = opaque_u32(ring0 + K6W * K6_ROWRING + warp * K6_QN * (uint32_t)M - (uint32_t)(M / 4) * qr);
    const uint32_t lt = opaque_u32((1u << lane) - 1u), tau = a.tau;
    if (threadIdx.x == 0) {
        mbar_init(&lut_bar, 1);
        fence_mbar_init();
    }
    const uint32_t nunits = min(*a.nitems, a.items_cap);
    uint32_t phase = 0;
    // ring head / tail in bytes of the row words (wrapping counters); survivors pushed so far
    uint32_t qh = 0, qt = 0, surv_n = 0;
    // Units are claimed two ahead by thread 0 and their items fetched one ahead, both while the
    // current unit is scanned (unit_s / item_s double-buffered by parity): a unit starts with
    // no dependent global loads.  u_nxt / it_nxt: the next unit and its item (thread 0 only).
    uint32_t u_nxt = 0;
    uint4 it_nxt = make_uint4(0u, 0u, 0u, 0u);
    if (threadIdx.x == 0) {
        const uint32_t u0 = atomicAdd(a.work, 1u);
        u_nxt = atomicAdd(a.work, 1u);
        unit_s[0] = u0;
        if (u0 < nunits) item_s[0] = __ldg(a.items + u0);
        if (u_nxt < nunits) it_nxt = __ldg(a.items + u_nxt);
    }
    for (uint32_t it = 0;; ++it) {
        __syncthreads();  // the previous unit's LUT and rings are no longer read; unit `it` is published
        const uint32_t u = unit_s[it & 1u];
        if (u >= nunits) break;
        const uint4 un = item_s[it & 1u];  // (query, probe, pos, rows)
        const uint32_t qi = un.x, item = un.x * a.nprobe + un.y;
        uint32_t u_nn = 0;
        if (threadIdx.x == 0) {  // the LUT by bulk copy; the barrier above ordered the prior generic reads
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&lut_bar, (uint32_t)(M * KSUB * 4));
            bulk_g2s(k6s, a.lutp + (size_t)item * M * KSUB, M * KSUB * 4, &lut_bar);
            u_nn = atomicAdd(a.work, 1u);  // unit it + 2; the value is not used before this unit ends
        }
        const C qc = reinterpret_cast<const C*>(a.qcodes)[item];
        const unsigned long long thr = __ldcg(a.thr + qi);
        const uint32_t n = un.w, pos0 = un.z;
        const C* ci = reinterpret_cast<const C*>(a.codes) + pos0;
        const uint32_t qt0 = qt;

        // drain cnt entries from the ring head (lanes < cnt busy)
        auto drain = [&](uint32_t cnt) {
            __syncwarp();
            if (lane < cnt) {
                const uint32_t ra = ((qh + 4u * lane) & (K6_ROWRING - 1u)) | qr;
                C cc;
                if constexpr (M == 8) {
                    const uint2 en = s_ld64((uint32_t)(M / 4) * ra + qk);
                    cc.x = en.x;
                    cc.y = en.y;
                } else {
                    cc = s_ld128((uint32_t)(M / 4) * ra + qk);
                }
                float score;
                if constexpr (STRAT == DUAL || STRAT == ADC) score = adc_sh<M>(lut0, cc, (uint32_t)(thr >> 32));
                else if constexpr (STRAT == BINARY) score = (float)ham(cc, qc);
                else score = (float)disidx(cc, qc);
                const uint32_t sb = __float_as_uint(score);
                if (sb <= (uint32_t)(thr >> 32)) {
                    const uint32_t row = s_ld32(ra);  // the row word is read only here
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
        // test 32 rows (one per lane) and push the survivors at the ring tail
        auto step = [&](const C& cv, uint32_t row, bool valid) {
            bool pass = valid;
            if constexpr (STRAT == DUAL) pass = pass && ham(cv, qc) <= tau;
            if constexpr (PERQ && (STRAT == DUAL || STRAT == ADC)) {  // stats mode: per-query count + id hash
                if (pass) {
                    atomicAdd(a.surv_q + qi, 1ull);
                    atomicAdd(a.hash_q + qi, (unsigned long long)mix64(__ldg(a.low + pos0 + row)));
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, pass);
            if (bal) {
                const uint32_t ra = ((qt + 4u * __popc(bal & lt)) & (K6_ROWRING - 1u)) | qr;
                s_st32_if(ra, row, pass);
                if constexpr (M == 8) s_st64_if((uint32_t)(M / 4) * ra + qk, cv.x, cv.y, pass);
                else s_st128_if((uint32_t)(M / 4) * ra + qk, cv.x, cv.y, cv.z, cv.w, pass);
                qt += 4u * __popc(bal);
            }
        };
        // 128 rows per warp block (4 per lane), drained after every 64
        auto block = [&](const C (&c)[4], uint32_t rb) {
            const uint32_t row0 = rb + lane;
            if (rb + 128u <= n) {  // a whole block: no row bound tests
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    step(c[2 * h], row0 + 64u * h, true);
                    step(c[2 * h + 1], row0 + 64u * h + 32u, true);
                    while (qt - qh >= 32u * 4u) {
                        drain(32);
                        qh += 32u * 4u;
                    }
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    step(c[2 * h], row0 + 64u * h, row0 + 64u * h < n);
                    step(c[2 * h + 1], row0 + 64u * h + 32u, row0 + 64u * h + 32u < n);
                    while (qt - qh >= 32u * 4u) {
                        drain(32);
                        qh += 32u * 4u;
                    }
                }
            }
        };
        // the next block's codes are loaded before this block is tested and drained; two
        // register sets alternate (no copies)
        auto load = [&](C (&c)[4], uint32_t rb) {
            const C* p = ci + rb + lane;
            if (rb + 128u <= n) {
#pragma unroll
                for (int v = 0; v < 4; ++v) c[v] = ld_stream(p + 32 * v);
            } else {
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    if (rb + 32u * v + lane < n) c[v] = ld_stream(p + 32 * v);
            }
        };
        constexpr uint32_t STRIDE = 128u * K6W;
        C ca[4], cb[4];
        uint32_t rb = warp * 128u;
        if (rb < n) load(ca, rb);  // in flight while the LUT arrives
        if (threadIdx.x == 0 && u_nxt < nunits) {
            // the next unit's codes and LUT are pulled into L2 now (one bulk prefetch each): when that
            // unit starts, its loads are L2 hits -- the bytes a warp keeps in flight no longer bound the scan
            const uintptr_t p0 = reinterpret_cast<uintptr_t>(a.codes) + (size_t)it_nxt.z * M;
            const uintptr_t lo = p0 & ~(uintptr_t)15, hi = (p0 + (size_t)it_nxt.w * M + 15) & ~(uintptr_t)15;
            bulk_prefetch_l2(reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo));
            if constexpr (STRAT == DUAL || STRAT == ADC)
                bulk_prefetch_l2(a.lutp + (size_t)(it_nxt.x * a.nprobe + it_nxt.y) * M * KSUB, (uint32_t)(M * KSUB * 4));
        }
        mbar_wait(&lut_bar, phase);
        phase ^= 1u;
        while (rb < n) {
            if (rb + STRIDE < n) load(cb, rb + STRIDE);
            block(ca, rb);
            rb += STRIDE;
            if (rb >= n) break;
            if (rb + STRIDE < n) load(ca, rb + STRIDE);
            block(cb, rb);
            rb += STRIDE;
        }
        if (qt != qh) {
            drain((qt - qh) >> 2);
            qh = qt;
        }
        if (threadIdx.x == 0) {  // publish unit it + 1 (its item was loaded during unit it - 1), fetch it + 2's
            unit_s[(it + 1u) & 1u] = u_nxt;
            item_s[(it + 1u) & 1u] = it_nxt;
            u_nxt = u_nn;
            if (u_nxt < nunits) it_nxt = __ldg(a.items + u_nxt);
        }
        if constexpr (STRAT == DUAL) {
            surv_n += (qt - qt0) >> 2;
            if (surv_n >= (1u << 30)) {  // keep the 32-bit count from wrapping
                if (lane == 0) atomicAdd(a.surv_total, (unsigned long long)surv_n);
                surv_n = 0;
            }
        }
    }
    if (STRAT == DUAL && lane == 0 && surv_n) atomicAdd(a.surv_total, (unsigned long long)surv_n);
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
