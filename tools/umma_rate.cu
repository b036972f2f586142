// Microbenchmark: issue rate and round-trip latency of tcgen05.mma for M = 128 and N in
// {16, 32, 64, 128, 256}, one CTA per SM: kind::i8 with A in TMEM (K = 32, K2's filter),
// kind::i8 with A in shared memory, and kind::mxf4 block-scaled e2m1 (K = 64, A and B in
// shared memory, unit scale factors in TMEM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_rate tools/umma_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N, int KIND>  // 0: i8 A in TMEM, 1: i8 A in smem, 2: mxf4
__global__ void rate(int rounds, int per_round, unsigned long long* out) {
    __shared__ __align__(1024) int8_t B[256 * 32 * 3];
    __shared__ __align__(1024) int8_t A[128 * 32 * 3];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (int)sizeof(B); i += blockDim.x) B[i] = (int8_t)(i * 7);
    for (int i = threadIdx.x; i < (int)sizeof(A); i += blockDim.x) A[i] = (int8_t)(i * 5);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tmem_base;
    // B K-major no swizzle: core (n8, k16) at n8 * 128 + k16 * (N * 16): LBO = 16 N, SBO = 128
    const uint32_t lbo = N * 16, sbo = 128;
    const uint64_t bdesc = (uint64_t)((smem_u32(B) & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) |
                           ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
    const uint32_t idesc = KIND == 2
        ? ((1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24))  // mxf4 e2m1, ue8m0
        : ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24));
    const uint32_t a_t = tm, d_t = tm + 256;  // A: 8 columns per K block; D: N columns
    const uint64_t adesc = (uint64_t)((smem_u32(A) & 0x3FFFFu) >> 4) | ((uint64_t)(2048u >> 4) << 16) |
                           ((uint64_t)(128u >> 4) << 32) | (1ull << 46);
    const uint32_t sfa = tm + 32, sfb = tm + 40;  // unit scale factors (ue8m0 127) in every byte
    if (KIND == 2) {
        const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                         sfa + lane_base), "r"(0x7F7F7F7Fu)
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    uint32_t phase = 0;
    unsigned long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            for (int i = 0; i < per_round; ++i) {
                const uint32_t acc = i > 0;
                if (KIND == 0)
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_t),
                        "r"(a_t + 8 * (i % 3)), "l"(bdesc + (uint64_t)(32 * (i % 3))), "r"(idesc), "r"(acc)
                        : "memory");
                else if (KIND == 1)
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_t),
                        "l"(adesc + (uint64_t)(2 * (i % 3))), "l"(bdesc + (uint64_t)(32 * (i % 3))), "r"(idesc), "r"(acc)
                        : "memory");
                else
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d_t),
                        "l"(adesc + (uint64_t)(2 * (i % 3))), "l"(bdesc + (uint64_t)(32 * (i % 3))), "r"(idesc), "r"(acc),
                        "r"(sfa), "r"(sfb)
                        : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&bar))
                         : "memory");
            asm volatile(
                "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                    smem_u32(&bar)),
                "r"(phase)
                : "memory");
            phase ^= 1;
        }
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int KIND>
void run(unsigned long long* d, int sms) {
    unsigned long long h[256];
    for (int per : {1, 6, 48}) {
        const int rounds = 4096 / per * 8;
        rate<N, KIND><<<sms, 128>>>(rounds, per, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += (double)h[i];
        avg /= sms;
        printf("%s N=%3d  %2d MMAs per commit+wait: %7.1f clk per round, %6.1f clk per MMA\n",
               KIND == 0 ? "i8 A-tmem" : (KIND == 1 ? "i8 A-smem" : "mxf4 K64 "), N, per, avg / rounds,
               avg / rounds / per);
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, 256 * 8);
    run<16, 0>(d, sms);
    run<128, 0>(d, sms);
    run<16, 1>(d, sms);
    run<128, 1>(d, sms);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    run<16, 2>(d, sms);
    run<32, 2>(d, sms);
    run<128, 2>(d, sms);
    const cudaError_t e = cudaGetLastError();
    printf("%s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    return 0;
}
