// Microbenchmark: the sq_l2 inner loop (sub, mul, add in dim order, no FMA contraction)
// as scalar FADD/FMUL vs packed f32x2 (FADD2 sub, FFMA2 t*t + z with z a runtime +0.0
// so ptxas cannot contract the square into the add, FADD2 add).  Checks bit equality.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32x2_bench tools/fp32x2_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}

// each thread: 16 "centroids" (register codebook), NR residual rows from smem, out = sums
template <bool PACKED>
__global__ void __launch_bounds__(256) k(const float* __restrict__ cb, const float* __restrict__ r, float z, int iters,
                                         float* __restrict__ out) {
    __shared__ __align__(16) float rs[8][16];
    if (threadIdx.x < 128) rs[threadIdx.x / 16][threadIdx.x % 16] = r[threadIdx.x];
    __syncthreads();
    float c[16];
    for (int d = 0; d < 16; ++d) c[d] = cb[(blockIdx.x * 256 + threadIdx.x) * 16 % 4096 + d];
    float sink = 0.f;
    for (int i = 0; i < iters; ++i) {
        if constexpr (!PACKED) {
            float acc[8];
#pragma unroll
            for (int it = 0; it < 8; ++it) acc[it] = 0.f;
#pragma unroll
            for (int d = 0; d < 16; ++d)
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const float t = __fsub_rn(rs[it][d], c[d]);
                    acc[it] = __fadd_rn(acc[it], __fmul_rn(t, t));
                }
#pragma unroll
            for (int it = 0; it < 8; ++it) sink += acc[it];
        } else {
            // pairs of items share a packed register: (item 2p, item 2p+1)
            unsigned long long acc[4];
            const unsigned long long zz = pk(z, z);
#pragma unroll
            for (int p = 0; p < 4; ++p) acc[p] = pk(0.f, 0.f);
#pragma unroll
            for (int d = 0; d < 16; ++d) {
                const unsigned long long cc = pk(c[d], c[d]);
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const unsigned long long x = pk(rs[2 * p][d], rs[2 * p + 1][d]);
                    unsigned long long t, s;
                    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(x), "l"(cc));
                    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s) : "l"(t), "l"(zz));
                    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc[p]) : "l"(acc[p]), "l"(s));
                }
            }
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                float a0, a1;
                upk(acc[p], a0, a1);
                sink += a0;
                sink += a1;
            }
        }
        c[i & 15] += 1e-7f;
    }
    out[blockIdx.x * 256 + threadIdx.x] = sink;
}

int main() {
    const int blocks = 148 * 8, iters = 2000;
    std::vector<float> hcb(4096 + 16), hr(128);
    for (size_t i = 0; i < hcb.size(); ++i) hcb[i] = (float)((i * 2654435761u) % 1000) * 0.01f;
    for (int i = 0; i < 128; ++i) hr[i] = (float)((i * 40503u) % 997) * 0.013f;
    float *cb, *r, *o0, *o1;
    cudaMalloc(&cb, hcb.size() * 4); cudaMalloc(&r, 512);
    cudaMalloc(&o0, blocks * 256 * 4); cudaMalloc(&o1, blocks * 256 * 4);
    cudaMemcpy(cb, hcb.data(), hcb.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(r, hr.data(), 512, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms[2];
    for (int v = 0; v < 2; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) k<false><<<blocks, 256>>>(cb, r, 0.0f, iters, o0);
            else k<true><<<blocks, 256>>>(cb, r, 0.0f, iters, o1);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms[v], e0, e1);
        }
    }
    std::vector<float> a(blocks * 256), b(blocks * 256);
    cudaMemcpy(a.data(), o0, a.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), o1, b.size() * 4, cudaMemcpyDeviceToHost);
    const bool same = memcmp(a.data(), b.data(), a.size() * 4) == 0;
    const double elems = (double)blocks * 256 * iters * 8 * 16;  // (item, dim) terms
    printf("{\"scalar_ms\": %.3f, \"packed_ms\": %.3f, \"scalar_terms_per_clk_sm\": %.1f, \"packed_terms_per_clk_sm\": %.1f, \"bit_equal\": %s}\n",
           ms[0], ms[1], elems / (ms[0] * 1e-3) / 148 / 1.965e9, elems / (ms[1] * 1e-3) / 148 / 1.965e9,
           same ? "true" : "false");
    return same ? 0 : 1;
}
