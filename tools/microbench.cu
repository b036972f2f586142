// Microbenchmarks that pin the roofline constants used in DESIGN.md:
// POPC issue rate, ALU (LOP3) rate, random shared-memory gather rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void popc_kernel(const uint32_t* __restrict__ in, uint32_t* out, int iters) {
    uint32_t a[8];
    #pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = in[(threadIdx.x + i) & 255] ^ (blockIdx.x * 2654435761u);
    uint32_t acc[8] = {0,0,0,0,0,0,0,0};
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int i = 0; i < 8; ++i) { acc[i] += __popc(a[i] ^ acc[(i + 1) & 7]); }
    }
    uint32_t s = 0;
    #pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 0xdeadbeef) out[0] = s;
}

__global__ void lop_kernel(const uint32_t* __restrict__ in, uint32_t* out, int iters) {
    uint32_t a[8];
    #pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = in[(threadIdx.x + i) & 255] ^ (blockIdx.x * 2654435761u);
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int i = 0; i < 8; ++i) { a[i] = (a[i] ^ a[(i + 1) & 7]) + 0x9e3779b9u; }
    }
    uint32_t s = 0;
    #pragma unroll
    for (int i = 0; i < 8; ++i) s ^= a[i];
    if (s == 0xdeadbeef) out[0] = s;
}

// random gathers from an 8 KB (2048-float) table per CTA, like one query's LUT
__global__ void lds_gather_kernel(float* out, int iters) {
    __shared__ float lut[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) lut[i] = (float)i;
    __syncthreads();
    uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int m = 0; m < 8; ++m) {
            x = x * 1664525u + 1013904223u;
            acc += lut[m * 256 + (x >> 24)];
        }
    }
    if (acc == -1.f) out[0] = acc;
}

// packed FP32: add.rn.f32x2 (FADD2), 8 independent chains per thread
__global__ void f32x2_kernel(const float* __restrict__ in, float* out, int iters) {
    unsigned long long a[8], b;
    const float x = in[threadIdx.x & 255], y = in[(threadIdx.x + 1) & 255];
    asm("mov.b64 %0, {%1,%2};" : "=l"(b) : "f"(x), "f"(y));
#pragma unroll
    for (int i = 0; i < 8; ++i) asm("mov.b64 %0, {%1,%2};" : "=l"(a[i]) : "f"(x + i), "f"(y - i));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(b));
    }
    unsigned long long s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= a[i];
    if (s == 0x1234567ull) out[0] = 1.f;
}

int main() {
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"name\":\"%s\",\"sm\":%d,\"l2\":%d,\"smem_optin\":%zu,\"smem_per_sm\":%zu,\"regs_per_sm\":%d,\"hbm_bytes\":%zu,\"clock_khz\":%d,\"cc\":\"%d.%d\"}\n",
           p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor,
           p.regsPerMultiprocessor, p.totalGlobalMem, clk, p.major, p.minor);
    uint32_t* d_in; uint32_t* d_out; float* d_f;
    CK(cudaMalloc(&d_in, 1024 * 4)); CK(cudaMalloc(&d_out, 1024 * 4)); CK(cudaMalloc(&d_f, 1024 * 4));
    CK(cudaMemset(d_in, 0x5a, 1024 * 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); popc_kernel<<<blocks, threads>>>(d_in, d_out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * iters * 8;
        printf("{\"bench\":\"popc\",\"ms\":%.3f,\"popc_per_s\":%.4e,\"popc_per_clk_sm_at_maxclk\":%.2f}\n", ms, ops / (ms * 1e-3),
               ops / (ms * 1e-3) / (p.multiProcessorCount * (clk * 1e3)));
        cudaEventRecord(e0); lop_kernel<<<blocks, threads>>>(d_in, d_out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        ops = (double)blocks * threads * iters * 8 * 2;
        printf("{\"bench\":\"lop+iadd\",\"ms\":%.3f,\"ops_per_s\":%.4e,\"ops_per_clk_sm_at_maxclk\":%.2f}\n", ms, ops / (ms * 1e-3),
               ops / (ms * 1e-3) / (p.multiProcessorCount * (clk * 1e3)));
        cudaEventRecord(e0); f32x2_kernel<<<blocks, threads>>>(reinterpret_cast<const float*>(d_in), d_f, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        ops = (double)blocks * threads * iters * 8 * 2;  // two fp32 adds per FADD2
        printf("{\"bench\":\"f32x2_add\",\"ms\":%.3f,\"fp32_ops_per_s\":%.4e,\"fp32_ops_per_clk_sm_at_maxclk\":%.2f}\n", ms, ops / (ms * 1e-3),
               ops / (ms * 1e-3) / (p.multiProcessorCount * (clk * 1e3)));
        cudaEventRecord(e0); lds_gather_kernel<<<blocks, threads>>>(d_f, iters / 4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        ops = (double)blocks * threads * (iters / 4) * 8;
        printf("{\"bench\":\"lds_random_gather\",\"ms\":%.3f,\"gathers_per_s\":%.4e,\"gathers_per_clk_sm_at_maxclk\":%.2f}\n", ms, ops / (ms * 1e-3),
               ops / (ms * 1e-3) / (p.multiProcessorCount * (clk * 1e3)));
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
