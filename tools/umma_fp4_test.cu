// Microtest of K2t's filter formulation (kernels_scan_tc.cu): one quad (128 codes) x 16
// queries through ONE block-scaled e2m1 MMA (kind::mxf4, K = 64) with A and B in shared
// memory, unit ue8m0 scale factors in TMEM and the accumulator preloaded with the bias
// |q| - tau - 1/2.  Checks D[code][q] == ham(code, q) - tau - 1/2 exactly.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_fp4_test tools/umma_fp4_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const uint2* codes, const uint2* qcodes, int tau, float* dout, int sf_col, int sfb_off) {
    __shared__ __align__(1024) uint8_t A[128 * 32];
    __shared__ __align__(1024) uint8_t B[16 * 32];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // B row n: element 8 (4 cw + sh) + i = bit 32 cw + 4 i + sh -> e2m1 +2 (0x4) / -2 (0xC)
    if (threadIdx.x < 128) {
        const uint32_t n = threadIdx.x >> 3, wd = threadIdx.x & 7u, cw = wd >> 2, sh = wd & 3u;
        const uint32_t q = cw ? qcodes[n].y : qcodes[n].x;
        const uint32_t v = 0x44444444u | (((q >> sh) & 0x11111111u) << 3);
        const uint32_t byte = wd * 4;
        *reinterpret_cast<uint32_t*>(B + (n >> 3) * 128 + (byte >> 4) * 256 + (n & 7) * 16 + (byte & 15)) = v;
    }
    // A row r: element 8 (4 cw + sh) + i = bit 32 cw + 4 i + sh -> 0.5 (0x1) / 0
    const uint32_t r = threadIdx.x;
    const uint2 c = codes[r];
    uint32_t w[8];
    for (int sh = 0; sh < 4; ++sh) {
        w[sh] = (c.x >> sh) & 0x11111111u;
        w[4 + sh] = (c.y >> sh) & 0x11111111u;
    }
    *reinterpret_cast<uint4*>(A + r * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(A + 2048 + r * 16) = make_uint4(w[4], w[5], w[6], w[7]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tmem_base;
    const uint32_t tl = (uint32_t)(32 * warp) << 16;
    // scale factors 1.0 everywhere in columns [sf_col, sf_col + 32)
    for (int col = 0; col < 32; col += 8)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tm + tl + sf_col + col),
                     "r"(0x7F7F7F7Fu)
                     : "memory");
    // accumulator (column 64..79) preloaded with |q| - tau - 1/2
    uint32_t bb[16];
    for (int q = 0; q < 16; ++q)
        bb[q] = __float_as_uint((float)(__popc(qcodes[q].x) + __popc(qcodes[q].y)) - (float)tau - 0.5f);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            tm + tl + 64),
        "r"(bb[0]), "r"(bb[1]), "r"(bb[2]), "r"(bb[3]), "r"(bb[4]), "r"(bb[5]), "r"(bb[6]), "r"(bb[7]), "r"(bb[8]),
        "r"(bb[9]), "r"(bb[10]), "r"(bb[11]), "r"(bb[12]), "r"(bb[13]), "r"(bb[14]), "r"(bb[15])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint64_t adesc = (uint64_t)((smem_u32(A) & 0x3FFFFu) >> 4) | ((uint64_t)(2048u >> 4) << 16) |
                               ((uint64_t)(128u >> 4) << 32) | (1ull << 46);
        const uint64_t bdesc = (uint64_t)((smem_u32(B) & 0x3FFFFu) >> 4) | ((uint64_t)(256u >> 4) << 16) |
                               ((uint64_t)(128u >> 4) << 32) | (1ull << 46);
        const uint32_t idesc = (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
        asm volatile(
            "{\n.reg .pred p;\nsetp.eq.u32 p, 1, 1;\n"
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], p;\n}\n" ::"r"(tm + 64),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(tm + sf_col), "r"(tm + sf_col + sfb_off)
            : "memory");
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t d[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
          "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
        : "r"(tm + tl + 64));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 16; ++q) dout[r * 16 + q] = __uint_as_float(d[q]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
    (void)lane;
}

int main() {
    uint2 hc[128], hq[16];
    srand(7);
    auto r32 = []() { return ((uint32_t)rand() << 16) ^ (uint32_t)rand(); };
    for (auto& c : hc) c = make_uint2(r32(), r32());
    for (auto& q : hq) q = make_uint2(r32(), r32());
    hc[0] = hq[0];                    // h = 0
    hc[1] = make_uint2(~hq[1].x, ~hq[1].y);  // h = 64
    uint2 *dc, *dq;
    float* dd;
    cudaMalloc(&dc, sizeof(hc));
    cudaMalloc(&dq, sizeof(hq));
    cudaMalloc(&dd, 128 * 16 * 4);
    cudaMemcpy(dc, hc, sizeof(hc), cudaMemcpyHostToDevice);
    cudaMemcpy(dq, hq, sizeof(hq), cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 3; ++variant) {
        const int sf_col = variant == 0 ? 0 : 32, sfb = variant == 2 ? 8 : 16;
        const int tau = 24;
        k<<<1, 128>>>(dc, dq, tau, dd, sf_col, sfb);
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("variant %d (sf_col %d, sfb +%d): %s\n", variant, sf_col, sfb, cudaGetErrorString(e));
            return 1;
        }
        float hd[128 * 16];
        cudaMemcpy(hd, dd, sizeof(hd), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < 128; ++r)
            for (int q = 0; q < 16; ++q) {
                const int h = __builtin_popcount(hc[r].x ^ hq[q].x) + __builtin_popcount(hc[r].y ^ hq[q].y);
                const float want = (float)h - (float)tau - 0.5f;
                if (hd[r * 16 + q] != want) {
                    if (bad < 5) printf("  r %d q %d: got %g want %g (h %d)\n", r, q, hd[r * 16 + q], want, h);
                    ++bad;
                }
            }
        printf("variant %d (sf_col %d, sfb +%d): %d / %d wrong\n", variant, sf_col, sfb, bad, 128 * 16);
    }
    return 0;
}
