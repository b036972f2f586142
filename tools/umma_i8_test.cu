// Microtest: int8 tcgen05.mma with A in TMEM computing Hamming-threshold signs.
// 4 warps (one quad) = 128 rows (codes), N = 16 queries, K = 64 code bits + 32 bias.
// Each lane expands its 64-bit code into weighted bit-planes (A rows), the
// queries' +-2^(6-j) weights + bias row live in smem (B, K-major, no swizzle).
// D[row][q] should equal 64 * (ham(code,q) - tau) - 32.
// Tries descriptor variants (LBO/SBO swapped) and reports which one is right.
// Also probes M = 64 with A rows in lanes 0-63: on B200 only rows 0-15 of each
// 32-lane quadrant come back right, i.e. an M = 64 MMA spans 16 lanes of every
// quadrant and still needs all four warps (no smaller MMA group for K2).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void expand_word(uint32_t w, uint32_t* out) {
#pragma unroll
    for (int j = 0; j < 7; ++j) out[j] = w & (0x01010101u << j);
    out[7] = (w >> 7) & 0x01010101u;
}

__global__ void k(const uint2* codes, const uint2* qcodes, int tau, int lbo, int sbo, int* dout, int MM) {
    __shared__ __align__(1024) int8_t B[16 * 96];  // built in the canonical layout below
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // B: element (n, k) for n < 16 queries, k < 96.  k < 64: code word k/32, plane j = (k%32)/4, byte t = k%4
    // -> code bit 32*(k/32) + 8t + j; weight = sgn * (j < 7 ? 2^(6-j) : 64).  k >= 64: bias block.
    // Canonical no-swizzle K-major: core matrix = 8 rows x 16 bytes (row stride 16 B);
    // core (n8, k16) at byte offset n8 * SBOb + k16 * LBOb.  (LBOb, SBOb given in bytes.)
    for (int idx = threadIdx.x; idx < 16 * 96; idx += blockDim.x) {
        const int n = idx / 96, kk = idx % 96;
        int v;
        if (kk < 64) {
            const int wsel = kk / 32, j = (kk % 32) / 4, t = kk % 4;
            const uint32_t qw = wsel ? qcodes[n].y : qcodes[n].x;
            const int qb = (qw >> (8 * t + j)) & 1;
            const int mag = j < 7 ? (1 << (6 - j)) : 64;
            v = qb ? -mag : mag;
        } else {
            // A bias elements are 2: sum over 32 entries = T / 2, T = 64 * (|q| - tau) - 32
            const int pc = __popc(qcodes[n].x) + __popc(qcodes[n].y);
            const int T = 32 * (pc - tau) - 16;
            const int e = kk - 64;
            const int base = T / 32, rem = T - base * 32;  // rem in (-32, 32)
            v = base + (e < (rem < 0 ? -rem : rem) ? (rem < 0 ? -1 : 1) : 0);
        }
        const int n8 = n / 8, r = n % 8, k16 = kk / 16, c = kk % 16;
        B[n8 * sbo + k16 * lbo + r * 16 + c] = (int8_t)v;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tmem_base;
    // A at columns [0, 24): 16 code columns + 8 bias columns (all ones); D at columns [32, 48)
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
    uint2 c = codes[threadIdx.x];
    uint32_t a[24];
    expand_word(c.x, a);
    expand_word(c.y, a + 8);
#pragma unroll
    for (int i = 16; i < 24; ++i) a[i] = 0x02020202u;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tm + lane_base + 0), "r"(a[0]),
        "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tm + lane_base + 8), "r"(a[8]),
        "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tm + lane_base + 16), "r"(a[16]),
        "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        // instruction descriptor: D s32 (2) bits 4-5; A s8 (1) bits 7-9; B s8 (1) bits 10-12; K-major both;
        // N >> 3 at bits 17-22; M >> 4 at bits 24-28
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | (((uint32_t)MM >> 4) << 24);
        for (int kb = 0; kb < 3; ++kb) {
            const uint32_t baddr = smem_u32(B) + kb * 2 * lbo;  // K block of 32 bytes = 2 core columns
            uint64_t desc = ((uint64_t)((baddr & 0x3FFFF) >> 4)) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                            ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
            const uint32_t a_t = tm + kb * 8, d_t = tm + 32;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_t),
                "r"(a_t), "l"(desc), "r"(idesc), "r"(kb));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    __syncwarp();
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t d[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
          "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
        : "r"(tm + lane_base + 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int q = 0; q < 16; ++q) dout[threadIdx.x * 16 + q] = (int)d[q];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(64));
}

int main() {
    std::vector<uint2> codes(128), q(16);
    srand(7);
    auto r32 = [] { return (uint32_t)rand() ^ ((uint32_t)rand() << 15) ^ ((uint32_t)rand() << 30); };
    for (auto& c : codes) c = make_uint2(r32(), r32());
    for (auto& c : q) c = make_uint2(r32(), r32());
    q[3] = make_uint2(0, 0);
    q[5] = make_uint2(~0u, ~0u);
    codes[9] = q[2];
    uint2 *dc, *dq;
    int* dd;
    cudaMalloc(&dc, 128 * 8);
    cudaMalloc(&dq, 16 * 8);
    cudaMalloc(&dd, 128 * 16 * 4);
    cudaMemcpy(dc, codes.data(), 128 * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, q.data(), 16 * 8, cudaMemcpyHostToDevice);
    const int variants[1][2] = {{256, 128}};  // (LBO bytes, SBO bytes)
    for (int MMv : {128, 64})
    for (int tau : {24, 0, 64}) {
        for (auto& v : variants) {
            cudaMemset(dd, 0, 128 * 16 * 4);
            k<<<1, 128>>>(dc, dq, tau, v[0], v[1], dd, MMv);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("lbo %d sbo %d: %s\n", v[0], v[1], cudaGetErrorString(e));
                return 1;
            }
            std::vector<int> h(128 * 16);
            cudaMemcpy(h.data(), dd, h.size() * 4, cudaMemcpyDeviceToHost);
            int bad = 0, first = -1;
            int badrows[4] = {0, 0, 0, 0};
            for (int r = 0; r < MMv; ++r)
                for (int n = 0; n < 16; ++n) {
                    const int ham = __builtin_popcount(codes[r].x ^ q[n].x) + __builtin_popcount(codes[r].y ^ q[n].y);
                    const int want = 64 * (ham - tau) - 32;
                    if (h[r * 16 + n] != want) {
                        if (first < 0) first = r * 16 + n;
                        ++bad;
                        ++badrows[r / 32];
                    }
                }
            printf("M %d tau %d: bad %d / %d (per quadrant %d %d %d %d)", MMv, tau, bad, MMv * 16, badrows[0], badrows[1], badrows[2], badrows[3]);
            if (first >= 0) {
                const int r = first / 16, n = first % 16;
                const int ham = __builtin_popcount(codes[r].x ^ q[n].x) + __builtin_popcount(codes[r].y ^ q[n].y);
                printf("  first r %d n %d got %d want %d", r, n, h[first], 64 * (ham - tau) - 32);
            }
            printf("\n");
        }
    }
    return 0;
}
