// code_ops.cuh -- per-code device arithmetic shared by the scan kernels (K2 flat,
// K6 IVF, the rescue scans): Hamming distance, disidx, the ADC sum and the
// survivor hash.  dbits = 8, so sub-quantizer field sq is byte sq of the code
// (code_get_field pq.hpp:22-43).
#pragma once

#include "poly_b200.cuh"

namespace pb {

template <int M> struct CodeT;
template <> struct CodeT<8> { using T = uint2; };
template <> struct CodeT<16> { using T = uint4; };

// hamming_bytes (flat_index.hpp:14-27): popcount of the xor, word by word
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
template <class C>
__device__ __forceinline__ uint32_t field(const C& c, int sq) {
    return (word(c, sq >> 2) >> (8 * (sq & 3))) & 0xFFu;
}

// adc_distance (pq.cpp:121-128) through a stored-field LUT (permuted_lut,
// pq.cpp:107-119): acc = 0; acc += L[sq][field_sq] in sq order (0 + x == x, x >= +0).
template <int M, class C>
__device__ __forceinline__ float adc(const float* __restrict__ L, const C& c) {
    float acc = L[field(c, 0)];
#pragma unroll
    for (int sq = 1; sq < M; ++sq) acc = __fadd_rn(acc, L[sq * KSUB + field(c, sq)]);
    return acc;
}

// Same with an exact early exit: the first M/2 terms in sq order; partial sums of
// non-negative terms under round-to-nearest are monotone, so a prefix above the
// bound's score makes the full sum exceed it too (+inf: never a candidate).
template <int M, class C>
__device__ __forceinline__ float adc_bounded(const float* L, const C& c, uint32_t bound_bits) {
    float acc = L[field(c, 0)];
#pragma unroll
    for (int sq = 1; sq < M / 2; ++sq) acc = __fadd_rn(acc, L[sq * KSUB + field(c, sq)]);
    if (__float_as_uint(acc) > bound_bits) return __int_as_float(0x7f800000);
#pragma unroll
    for (int sq = M / 2; sq < M; ++sq) acc = __fadd_rn(acc, L[sq * KSUB + field(c, sq)]);
    return acc;
}

// Score of one code under a strategy (flat_index.hpp:44); false
// when the dual strategy's Hamming filter rejects the code (h > tau).
template <int M, int STRAT, class C>
__device__ __forceinline__ bool strategy_score(const float* L, const C& code, const C& qc, uint32_t tau,
                                               uint32_t bound_bits, float& score) {
    if constexpr (STRAT == DUAL) {
        if (ham(code, qc) > tau) return false;
        score = adc_bounded<M>(L, code, bound_bits);
    } else if constexpr (STRAT == ADC) {
        score = adc_bounded<M>(L, code, bound_bits);
    } else if constexpr (STRAT == BINARY) {
        score = (float)ham(code, qc);
    } else {
        score = (float)disidx(code, qc);
    }
    return true;
}

}  // namespace pb
