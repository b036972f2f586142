// scan_common.cuh -- device helpers shared by the flat scan kernels (K2 in
// kernels_scan.cu, the role-split tensor-core K2 in kernels_scan_tc.cu): key words,
// shared-window accesses, the ADC sums, the tensor-core filter's operand layout and
// the candidate append with its threshold-select request ring.
#pragma once

#include "code_ops.cuh"

namespace pb {

__device__ __forceinline__ uint32_t key_low(const ScanArgs& a, uint32_t pos) {
    return a.id_mode == ID_ARITH ? a.id0 + pos : __ldg(a.id32 + pos);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Explicit shared-window accesses on 32-bit addresses: keeps the hot loop free
// of generic-pointer materialisation (S2R SR_CgaCtaId + LEA per access).
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds32v(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ float ldsf(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void lds_code(uint32_t addr, uint2& c) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(c.x), "=r"(c.y) : "r"(addr));
}
__device__ __forceinline__ void lds_code(uint32_t addr, uint4& c) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "r"(addr));
}

// ADC from a query's stored-field LUT at shared address L (bytes), in sq order.
template <int M, class C>
__device__ __forceinline__ float adc_s(uint32_t L, const C& c) {
    float acc = ldsf(L + 4u * (word(c, 0) & 0xFFu));
#pragma unroll
    for (int sq = 1; sq < M; ++sq) {
        const uint32_t f = (word(c, sq >> 2) >> (8 * (sq & 3))) & 0xFFu;
        acc = __fadd_rn(acc, ldsf(L + 4u * (sq * KSUB + f)));
    }
    return acc;
}

// ADC with an exact early exit: the first M/2 terms are summed in sq order;
// partial sums of non-negative terms with round-to-nearest are monotone, so if
// that prefix already exceeds the bound's score the full sum does too and the
// pair can never become a candidate (returns +inf, no further LUT traffic).
template <int M, class C>
__device__ __forceinline__ float adc_s_bounded(uint32_t L, const C& c, uint32_t bound_bits) {
    float acc = ldsf(L + 4u * (word(c, 0) & 0xFFu));
#pragma unroll
    for (int sq = 1; sq < M / 2; ++sq) {
        const uint32_t f = (word(c, sq >> 2) >> (8 * (sq & 3))) & 0xFFu;
        acc = __fadd_rn(acc, ldsf(L + 4u * (sq * KSUB + f)));
    }
    if (__float_as_uint(acc) > bound_bits) return __int_as_float(0x7f800000);
#pragma unroll
    for (int sq = M / 2; sq < M; ++sq) {
        const uint32_t f = (word(c, sq >> 2) >> (8 * (sq & 3))) & 0xFFu;
        acc = __fadd_rn(acc, ldsf(L + 4u * (sq * KSUB + f)));
    }
    return acc;
}

// Four Hamming distances (each <= 128) packed into the bytes of one word.
template <class C>
__device__ __forceinline__ uint32_t ham4(const C& code, const C* qc) {
    const uint32_t h0 = ham(code, qc[0]), h1 = ham(code, qc[1]), h2 = ham(code, qc[2]), h3 = ham(code, qc[3]);
    return (h0 + (h1 << 8)) + ((h2 + (h3 << 8)) << 16);
}

// ---- tensor-core Hamming filter (DUAL) ----
// h(x, q) <= tau is decided by one int8 MMA per 128 codes x 16 queries: code bit b of
// byte t of word w becomes A element (w, plane j = b, byte t) with value 2^j (j < 7) or
// 1 (j = 7) -- one LOP per 4 elements; the query's B element is s * 64 / value with
// s = +1 / -1 for query bit 0 / 1, so the products sum to 64 * (|x| - 2<x,q>) =
// 64 * (h - |q|).  A bias K-block (A = 2, B summing to 32 (|q| - tau) - 16) makes
// D = 64 (h - tau) - 32, i.e. sign(D) = [h <= tau], exact for every tau in [0, 64 * m/8].
__device__ __forceinline__ void expand_word(uint32_t w, uint32_t* out) {
#pragma unroll
    for (int j = 0; j < 7; ++j) out[j] = w & (0x01010101u << j);
    out[7] = (w >> 7) & 0x01010101u;
}
// B operand: 16 rows (queries) x KB bytes, canonical K-major no-swizzle layout:
// 8 x 16-byte core matrices, core (n8, k16) at n8 * 128 + k16 * 256 (SBO 128, LBO 256)
__device__ __forceinline__ uint32_t bw_offset(uint32_t n, uint32_t k) {
    return (n >> 3) * 128u + (k >> 4) * 256u + (n & 7u) * 16u + (k & 15u);
}
__device__ __forceinline__ uint64_t bw_desc(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(256u >> 4) << 16) | ((uint64_t)(128u >> 4) << 32) |
           (1ull << 46);
}
// kind::i8 instruction descriptor: D s32, A s8, B s8, K-major, N = 16, M = 128
constexpr uint32_t IDESC_I8_M128_N16 = (2u << 4) | (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

// Append a candidate key for batch query qg; track block completion.
__device__ __forceinline__ void append_candidate(const ScanArgs& a, uint32_t qg, unsigned long long key, uint32_t bs,
                                                 uint32_t* nreq_s, uint32_t* req_s) {
    const uint32_t slot = atomicAdd(&a.ccount[qg], 1u);
    if (slot >= a.cap) {  // list full: the rescue scan (kernels_rescue.cu) re-ranks this query exactly
        a.ovq[qg] = 1u;
        return;
    }
    a.cand[(size_t)qg * a.cap + slot] = key;
    __threadfence();
    const uint32_t nblk = a.cap / bs;
    const uint32_t blk = slot / bs;
    if (atomicAdd(&a.bdone[(size_t)qg * nblk + blk], 1u) == bs - 1) {
        // request ring served by the producer warp; a full ring drops the request
        // (thresholds are an optimisation, never needed for correctness)
        const uint32_t r = atomicAdd(nreq_s, 1u);
        req_s[r % MAXREQ] = (qg << 16) | blk;
    }
}

__device__ __forceinline__ void try_candidate(const ScanArgs& a, uint32_t qg, float score, uint32_t pos,
                                              unsigned long long thr, uint32_t bs, uint32_t* nreq_s, uint32_t* req_s) {
    const uint32_t sb = __float_as_uint(score);
    if (sb <= (uint32_t)(thr >> 32)) {
        const unsigned long long key = ((unsigned long long)sb << 32) | key_low(a, pos);
        if (key < thr) append_candidate(a, qg, key, bs, nreq_s, req_s);
    }
}

// k-th smallest (1-based) of n distinct keys in global memory; one warp,
// 8-pass radix select over 8-bit digits, keys streamed from L2 each pass.
static __device__ unsigned long long warp_select_kth(const unsigned long long* src, uint32_t n, uint32_t kk, uint32_t* hist) {
    const int lane = threadIdx.x & 31;
    unsigned long long prefix = 0, mask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = lane; i < 256; i += 32) hist[i] = 0;
        __syncwarp();
#pragma unroll 16
        for (uint32_t i = lane; i < n; i += 32) {
            const unsigned long long v = __ldcg(src + i);
            if ((v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 0xFFu], 1u);
        }
        __syncwarp();
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
        const bool mine = excl < kk && kk <= incl;
        uint32_t r = kk - excl;
        int digit = lane * 8 + 7;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (r <= c[j]) { digit = lane * 8 + j; break; }
            r -= c[j];
        }
        const int src_lane = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        digit = __shfl_sync(0xffffffffu, digit, src_lane);
        kk = __shfl_sync(0xffffffffu, r, src_lane);
        prefix |= (unsigned long long)digit << shift;
        mask |= 0xFFull << shift;
        __syncwarp();
    }
    return prefix;
}

}  // namespace pb
