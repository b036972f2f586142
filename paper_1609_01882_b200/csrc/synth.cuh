// synth.cuh -- counter-based Gaussian-mixture generator, device side.
//
// Bit-identical twin of oracle/polyoracle.c po_gen_centers / po_gen_points:
// integer hashing (splitmix64 finaliser), an exact-rounding int64 -> fp32
// conversion and explicitly rounded IEEE adds/muls (no FMA contraction).
// N(0,1) is approximated by Irwin-Hall(12).  Stream ids: 0 centers,
// 1 train, 2 base, 3 queries.
#pragma once
#include <cstdint>

#include "poly_b200.cuh"  // mix64

namespace pb {

__host__ __device__ __forceinline__ uint64_t row_key(uint64_t seed, uint32_t stream, uint64_t row) {
    const uint64_t base = mix64(seed + 0x632BE59BD9B4E019ull * (uint64_t)(stream + 1));
    return mix64(base ^ (row * 0xD1B54A32D192ED03ull));
}

__device__ __forceinline__ float synth_normal(uint64_t rowkey, uint32_t t) {
    uint64_t s = 0;
#pragma unroll
    for (uint32_t j = 0; j < 6; ++j) {
        const uint64_t h = mix64(rowkey ^ ((uint64_t)(6u * t + j + 1u) * 0xA0761D6478BD642Full));
        s += (h >> 40) + ((h >> 16) & 0xFFFFFFull);
    }
    const long long c = (long long)s - 6ll * 16777216ll;
    return __fmul_rn(__ll2float_rn(c), 1.0f / 16777216.0f);
}

__device__ __forceinline__ uint32_t synth_center(uint64_t rowkey, uint32_t ncent) {
    return (uint32_t)(((mix64(rowkey ^ 0x5851F42D4C957F2Dull) >> 32) * (uint64_t)ncent) >> 32);
}

// x_t = max(0, C[u][t] + N(0,1))
__device__ __forceinline__ float synth_coord(const float* center_row, uint64_t rowkey, uint32_t t) {
    const float v = __fadd_rn(center_row[t], synth_normal(rowkey, t));
    return v > 0.0f ? v : 0.0f;
}

// 1 / ||x|| exactly as the oracle computes it (0 for the zero vector).
__device__ __forceinline__ float synth_inv_norm(const float* center_row, uint64_t rowkey, uint32_t dim) {
    float nrm = 0.0f;
    for (uint32_t t = 0; t < dim; ++t) {
        const float x = synth_coord(center_row, rowkey, t);
        nrm = __fadd_rn(nrm, __fmul_rn(x, x));
    }
    return nrm > 0.0f ? __fdiv_rn(1.0f, __fsqrt_rn(nrm)) : 0.0f;
}

}  // namespace pb
