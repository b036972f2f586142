// kernels_coarse.cu -- enumerate_cells on the tensor cores, exact.
//
// enumerate_cells ranks the nprobe cells with the smallest sq_l2(q, c) (distances.cpp:
// 10-17, fp32 in dimension order), ascending, ties to the lower cell.  The reference
// primitive for "nearest cells" is assign_nearest (distances.cpp:56-79: |x|^2 - 2 x.c +
// |c|^2 through a BLAS GEMM).  Here:
//
//   K5t  coarse_tc_kernel (tcgen05.mma kind::tf32, accumulators in TMEM): per tile of
//        128 queries x 256 cells, D = Q . C^T; the epilogue turns D into
//        a'(c) = |c|^2 - 2 q.c (= a(c) - |q|^2) and keeps, per (query, group of 128
//        cells), the three smallest a' with the cells of the two smallest.  Only these
//        16-byte records reach global memory -- the nq x nlist distance block never does.
//   K5q  coarse_rank_kernel, one CTA per query: T = an upper bound of the np-th smallest
//        a' over the kept values (distinct cells, so >= the np-th smallest over all
//        cells); every cell of the exact top-np has a'(c) <= T + 2E, where E bounds
//        |fl(sq_l2(q, c)) - (|q|^2 + a'(c))| (TF32 operands, fp32 accumulation, the
//        reference's own rounding); such cells are among a group's two kept cells
//        unless the group's third value is itself within the bound, in which case the
//        whole group is a candidate.  Candidates get the exact fp32 sq_l2 in dimension
//        order and are ranked by (dist bits << 32 | cell), so the probe order is
//        bit-identical to the reference's.
//
// Layouts (no swizzle, K-major canonical UMMA layout: 8-row x 16-byte core matrices,
// SBO = 128 B between 8-row groups, LBO = rows / 8 * 128 B between 4-element K chunks):
//   A (queries)  128 rows x dim, resident in shared memory for the CTA's query tile;
//   B (cells)    256 rows x 32 dims per 32 KB pipeline stage, streamed by 1-D bulk copies
//                from a pre-packed copy of the centroids (built once at index creation).
#include <algorithm>

#include "poly_b200.cuh"

namespace pb {

constexpr int CT_M = 128;              // queries per tile (TMEM lanes)
constexpr int CT_N = 256;              // cells per tile (TMEM columns per accumulator)
#ifndef POLY_CT_KC
#define POLY_CT_KC 32
#endif
#ifndef POLY_CT_SMEM  // dynamic shared memory budget of K5t (A + the B stages)
#define POLY_CT_SMEM (225 * 1024)
#endif
constexpr int CT_KC = POLY_CT_KC;       // dims per pipeline stage
constexpr int CT_STAGE = CT_N * CT_KC * 4;  // 32 KB at 32 dims
constexpr int CT_MAX_STAGES = 16;
constexpr int CT_EPI_WARPS = 8;        // two per TMEM lane quadrant, one per 128-cell group
constexpr int CT_THREADS = (2 + CT_EPI_WARPS) * 32;
constexpr int CT_GROUP = 128;          // cells per kept-value group
constexpr float CT_PAD_NORM = 3.0e38f;  // |c|^2 of a pad cell: above every real a', finite under the index packing

// tcgen05 kind::tf32 instruction descriptor: D fp32, A/B tf32, both K-major, N = 256, M = 128
constexpr uint32_t IDESC_TF32_M128_N256 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(CT_N >> 3) << 17) |
                                          ((uint32_t)(CT_M >> 4) << 24);

__device__ __forceinline__ uint64_t ct_desc(uint32_t saddr, uint32_t lbo) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(128u >> 4) << 32) |
           (1ull << 46);
}

__device__ __forceinline__ void mma_tf32_ss(uint32_t d_t, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_t),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------- packing (index creation)
// packed[t][s] = the 32 KB shared-memory image of cells [256 t, 256 t + 256) x dims
// [32 s, 32 s + 32); cnorm_pad[c] = |c|^2 (any rounding: E covers it), CT_PAD_NORM for pad cells.
__global__ void coarse_pack_kernel(const float* __restrict__ cent, uint32_t nlist, uint32_t dim, uint32_t ntiles,
                                   float* __restrict__ packed, float* __restrict__ cnorm_pad) {
    const uint32_t nchunk = dim / CT_KC;
    const uint64_t total4 = (uint64_t)ntiles * CT_N * dim / 4;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total4; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k4 = (uint32_t)(e % (dim / 4));
        const uint64_t cell = e / (dim / 4);
        const uint32_t t = (uint32_t)(cell / CT_N), row = (uint32_t)(cell % CT_N);
        const uint32_t s = k4 / (CT_KC / 4), kc = k4 % (CT_KC / 4);
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (cell < nlist) v = reinterpret_cast<const float4*>(cent + cell * dim)[k4];
        const size_t off = ((size_t)t * nchunk + s) * (CT_STAGE / 4) + ((size_t)kc * (CT_N / 8) + row / 8) * 32 +
                           (row % 8) * 4;
        *reinterpret_cast<float4*>(packed + off) = v;
    }
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < (uint64_t)ntiles * CT_N;
         c += (uint64_t)gridDim.x * blockDim.x) {
        float acc = 0.f;
        if (c < nlist)
            for (uint32_t d = 0; d < dim; ++d) acc = __fmaf_rn(cent[c * dim + d], cent[c * dim + d], acc);
        cnorm_pad[c] = c < nlist ? acc : CT_PAD_NORM;
    }
}

void launch_coarse_pack(const float* cent, uint32_t nlist, uint32_t dim, float* packed, float* cnorm_pad,
                        cudaStream_t s) {
    const uint32_t ntiles = (nlist + CT_N - 1) / CT_N;
    coarse_pack_kernel<<<592, 256, 0, s>>>(cent, nlist, dim, ntiles, packed, cnorm_pad);
    count_launch();
}

uint32_t coarse_tc_tiles(uint32_t nlist) { return (nlist + CT_N - 1) / CT_N; }

// ---------------------------------------------------------------- K5t
// grid = (slices, query tiles); CTA (s, qt) handles the cell tiles [T s / S, T (s + 1) / S)
// of query tile qt.  Warp 0: bulk-copy producer; warp 1: TMEM owner + MMA issuer (one
// thread); warps 2..9: epilogue (warp w reads TMEM lane quadrant w % 4, cell group (w - 2) / 4).
__global__ void __launch_bounds__(CT_THREADS, 1) coarse_tc_kernel(const float* __restrict__ q, uint32_t nq,
                                                                  uint32_t dim, const float* __restrict__ packed,
                                                                  const float* __restrict__ cnorm_pad, uint32_t ntiles,
                                                                  uint32_t stages, float4* __restrict__ grp) {
    extern __shared__ __align__(1024) uint8_t ct_smem[];
    __shared__ __align__(8) uint64_t full_bar[CT_MAX_STAGES], empty_bar[CT_MAX_STAGES], tfull[2], tempty[2];
    __shared__ uint32_t tmem_s;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t S = gridDim.x, s = blockIdx.x, qt = blockIdx.y;
    const uint32_t t0 = (uint32_t)((uint64_t)ntiles * s / S), t1 = (uint32_t)((uint64_t)ntiles * (s + 1) / S);
    const uint32_t nchunk = dim / CT_KC;
    uint8_t* A = ct_smem;                                   // CT_M x dim, 128 * dim * 4 bytes
    uint8_t* Bst = ct_smem + (size_t)CT_M * dim * 4;        // stages x 32 KB

    // A: queries of this tile into the canonical K-major layout (zero rows past nq)
    const uint32_t n4 = CT_M * dim / 4;
    for (uint32_t e = threadIdx.x; e < n4; e += CT_THREADS) {
        const uint32_t row = e / (dim / 4), k4 = e % (dim / 4);
        const uint32_t qi = qt * CT_M + row;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (qi < nq) v = __ldg(reinterpret_cast<const float4*>(q + (size_t)qi * dim) + k4);
        *reinterpret_cast<float4*>(A + ((size_t)k4 * (CT_M / 8) + row / 8) * 128 + (row % 8) * 16) = v;
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < stages; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&empty_bar[i], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], CT_EPI_WARPS);  // every epilogue warp reads buffer b
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&tmem_s, 2 * CT_N);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_s;
    const uint32_t nunits = t1 - t0;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t sc = 0;
            for (uint32_t u = 0; u < nunits; ++u)
                for (uint32_t c = 0; c < nchunk; ++c, ++sc) {
                    const uint32_t st = sc % stages;
                    if (sc >= stages) mbar_wait(&empty_bar[st], ((sc / stages) - 1) & 1u);
                    mbar_arrive_expect_tx(&full_bar[st], CT_STAGE);
                    bulk_g2s(Bst + (size_t)st * CT_STAGE, packed + ((size_t)(t0 + u) * nchunk + c) * (CT_STAGE / 4),
                             CT_STAGE, &full_bar[st]);
                }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t a0 = smem_u32(A), b0 = smem_u32(Bst);
            const uint32_t lbo_a = CT_M / 8 * 128, lbo_b = CT_N / 8 * 128;
            uint32_t sc = 0;
            for (uint32_t u = 0; u < nunits; ++u) {
                const uint32_t buf = u & 1u;
                if (u >= 2) mbar_wait(&tempty[buf], ((u / 2) - 1) & 1u);
                tc_fence_after();
                const uint32_t d = tbase + buf * CT_N;
                for (uint32_t c = 0; c < nchunk; ++c, ++sc) {
                    const uint32_t st = sc % stages;
                    mbar_wait(&full_bar[st], (sc / stages) & 1u);
                    tc_fence_after();
#pragma unroll
                    for (uint32_t kk = 0; kk < CT_KC / 8; ++kk) {  // K = 8 per MMA: two 4-element core chunks
                        const uint64_t ad = ct_desc(a0 + (c * (CT_KC / 4) + 2 * kk) * lbo_a, lbo_a);
                        const uint64_t bd = ct_desc(b0 + st * CT_STAGE + 2 * kk * lbo_b, lbo_b);
                        mma_tf32_ss(d, ad, bd, IDESC_TF32_M128_N256, (c | kk) != 0);
                    }
                    tc_commit(&empty_bar[st]);  // the stage is free once these MMAs have read it
                }
                tc_commit(&tfull[buf]);
            }
        }
    } else {
        const uint32_t quad = warp & 3u, half = (warp - 2) >> 2;
        const uint32_t row = quad * 32 + lane, qi = qt * CT_M + row;
        for (uint32_t u = 0; u < nunits; ++u) {
            const uint32_t buf = u & 1u;
            mbar_wait(&tfull[buf], (u / 2) & 1u);
            tc_fence_after();
            const uint32_t tile = t0 + u;
            const float* cn = cnorm_pad + (size_t)tile * CT_N + half * CT_GROUP;
            // Branch-free selection: the cell's index within the group rides in the low 7 mantissa
            // bits of a' (a relative perturbation <= 2^-16, covered by K5q's error bound E), so the
            // three smallest packed values -- four min/max per value, merged two values at a time --
            // carry their cells along and are always distinct.  Pad cells have |c|^2 = 3e38 (finite: no NaN from the packing).
            float m1 = __int_as_float(0x7f800000), m2 = m1, m3 = m1;
#pragma unroll 1
            for (uint32_t c0 = 0; c0 < CT_GROUP; c0 += 32) {
                float d[32];
                tmem_ld32(tbase + ((quad * 32u) << 16) + buf * CT_N + half * CT_GROUP + c0, d);
                tmem_wait_ld();
#pragma unroll
                for (uint32_t j4 = 0; j4 < 8; ++j4) {
                    const float4 n4v = __ldg(reinterpret_cast<const float4*>(cn + c0) + j4);  // uniform: broadcast
                    const float nv[4] = {n4v.x, n4v.y, n4v.z, n4v.w};
#pragma unroll
                    for (uint32_t e = 0; e < 4; e += 2) {
                        // two packed values at a time: the three smallest of {m1 <= m2 <= m3} U {lo <= hi}
                        const uint32_t j = c0 + 4 * j4 + e;
                        const float a = __fmaf_rn(-2.0f, d[4 * j4 + e], nv[e]);
                        const float b = __fmaf_rn(-2.0f, d[4 * j4 + e + 1], nv[e + 1]);
                        const float ap = __uint_as_float((__float_as_uint(a) & ~(CT_GROUP - 1u)) | j);
                        const float bp = __uint_as_float((__float_as_uint(b) & ~(CT_GROUP - 1u)) | (j + 1u));
                        const float lo = fminf(ap, bp), hi = fmaxf(ap, bp);
                        const float x = fmaxf(m1, lo);
                        m3 = fminf(fminf(m3, fmaxf(m2, lo)), fmaxf(m1, hi));
                        m2 = fminf(fminf(m2, x), hi);
                        m1 = fminf(m1, lo);
                    }
                }
            }
            const uint32_t i1 = __float_as_uint(m1) & (CT_GROUP - 1u), i2 = __float_as_uint(m2) & (CT_GROUP - 1u);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cta(&tempty[buf]);
            if (qi < nq)
                grp[((size_t)tile * 2 + half) * nq + qi] = make_float4(m1, m2, m3, __uint_as_float(i1 | (i2 << 16)));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, 2 * CT_N);
    }
}

size_t coarse_tc_smem(uint32_t dim, uint32_t* stages) {
    const size_t a = (size_t)CT_M * dim * 4;
    // as many stages as fit: the main loop is bound by the bulk copies' latency, i.e. by the bytes in flight
    uint32_t st = (uint32_t)std::min<size_t>(CT_MAX_STAGES, ((size_t)POLY_CT_SMEM - a) / CT_STAGE);
    if (stages) *stages = st;
    return a + (size_t)st * CT_STAGE;
}

void launch_coarse_tc(const float* q, uint32_t nq, uint32_t dim, const float* packed, const float* cnorm_pad,
                      uint32_t nlist, int num_sms, float4* grp, cudaStream_t s) {
    if (nq == 0) return;
    const uint32_t ntiles = coarse_tc_tiles(nlist), qtiles = (nq + CT_M - 1) / CT_M;
    uint32_t stages = 0;
    const size_t smem = coarse_tc_smem(dim, &stages);
    // grid = slices x query tiles: pick the slice count (each slice >= 8 cell tiles) whose last
    // wave is fullest -- with 79 query tiles (10,000 queries) one slice would leave 69 SMs idle
    uint32_t slices = 1;
    double best = 0.0;
    for (uint32_t sl = 1; sl <= std::max<uint32_t>(1, std::min<uint32_t>(ntiles / 8, 32)); ++sl) {
        const uint64_t ctas = (uint64_t)sl * qtiles, waves = (ctas + num_sms - 1) / num_sms;
        const double eff = (double)ctas / (double)(waves * (uint64_t)num_sms) - 0.002 * sl;  // mild bias to fewer
        if (eff > best + 1e-9) {
            best = eff;
            slices = sl;
        }
    }
    set_max_smem((const void*)coarse_tc_kernel, smem);
    coarse_tc_kernel<<<dim3(slices, qtiles), CT_THREADS, smem, s>>>(q, nq, dim, packed, cnorm_pad, ntiles, stages,
                                                                   grp);
    count_launch();
}

// ---------------------------------------------------------------- K5q
constexpr int CR_THREADS = 512, CR_CHUNK = 2048, CR_BUF = 4096;  // np + chunk <= buf (pow2)
constexpr uint32_t CR_RANKMAX = 1024;                             // rank by counting up to this many keys
uint32_t coarse_rank_npmax() { return 1024; }

__device__ __forceinline__ uint32_t cr_ord(float f) {  // order-preserving float -> uint32
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float cr_unord(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// One CTA per query: thread t merges the records of groups t, t + 512, ... into its
// three smallest a' (with the cells of the two smallest); T = the upper edge of the
// 16-bit radix bucket of the np-th smallest of those values; candidates a' <= T + 2E
// (a thread whose third value is within the bound contributes all its groups' cells);
// the exact fp32 sq_l2 of the candidates ranks them.
__global__ void __launch_bounds__(CR_THREADS, 2) coarse_rank_kernel(const float* __restrict__ q, uint32_t nq,
                                                                    uint32_t dim, const float4* __restrict__ grp,
                                                                    uint32_t ngroups, float cmax,
                                                                    const float* __restrict__ cent, uint32_t nlist,
                                                                    uint32_t np, uint32_t* __restrict__ scratch,
                                                                    unsigned long long* __restrict__ probe_keys,
                                                                    uint32_t* __restrict__ probe_counts) {
    extern __shared__ __align__(16) uint8_t cr_smem[];
    unsigned long long* buf = reinterpret_cast<unsigned long long*>(cr_smem);  // CR_BUF keys
    float* qs = reinterpret_cast<float*>(buf + CR_BUF);                         // dim
    __shared__ float red_f[CR_THREADS / 32];
    __shared__ uint32_t red_u[2];
    __shared__ uint32_t ncand_s;
    const uint32_t qi = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* qrow = q + (size_t)qi * dim;
    uint32_t* cand = scratch + (size_t)qi * nlist;
    float qn = 0.0f;
    for (uint32_t d = tid; d < dim; d += CR_THREADS) {
        const float v = qrow[d];
        qs[d] = v;
        qn += v * v;
    }
    for (int off = 16; off; off >>= 1) qn += __shfl_xor_sync(0xffffffffu, qn, off);
    if (lane == 0) red_f[warp] = qn;
    if (tid == 0) ncand_s = 0;
    __syncthreads();
    qn = 0.0f;
    for (int w = 0; w < CR_THREADS / 32; ++w) qn += red_f[w];
    // this thread's groups: the three smallest a' and the cells of the two smallest
    float m1 = __int_as_float(0x7f800000), m2 = m1, m3 = m1;
    uint32_t i1 = 0xFFFFFFFFu, i2 = 0xFFFFFFFFu;
    auto keep = [&](float a, uint32_t c) {
        if (a < m3) {
            if (a < m2) {
                m3 = m2;
                if (a < m1) { m2 = m1; i2 = i1; m1 = a; i1 = c; }
                else { m2 = a; i2 = c; }
            } else {
                m3 = a;
            }
        }
    };
    for (uint32_t g = tid; g < ngroups; g += CR_THREADS) {
        const float4 r = grp[(size_t)g * nq + qi];
        const uint32_t pk = __float_as_uint(r.w), base = g * CT_GROUP;
        if ((pk & 0xFFFFu) != 0xFFFFu) keep(r.x, base + (pk & 0xFFFFu));
        if ((pk >> 16) != 0xFFFFu) keep(r.y, base + (pk >> 16));
        if (r.z < m3) m3 = r.z;  // (r.z >= r.y >= r.x: only the third value can still matter)
    }
    // T: radix select of the np-th smallest kept value (top 16 bits)
    uint32_t* hist = reinterpret_cast<uint32_t*>(buf);
    const uint32_t k1 = cr_ord(m1), k2 = cr_ord(m2), k3 = cr_ord(m3);
    const uint32_t nkept = 3 * min(ngroups, (uint32_t)CR_THREADS);  // >= distinct kept values
    uint32_t prefix = 0, want = min(np, nkept);
    for (int pass = 0; pass < 2; ++pass) {
        const int sh = 24 - 8 * pass;
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
        const uint32_t pm = pass ? prefix >> (sh + 8) : 0;
        if (!pass || (k1 >> (sh + 8)) == pm) atomicAdd(&hist[(k1 >> sh) & 255u], 1u);
        if (!pass || (k2 >> (sh + 8)) == pm) atomicAdd(&hist[(k2 >> sh) & 255u], 1u);
        if (!pass || (k3 >> (sh + 8)) == pm) atomicAdd(&hist[(k3 >> sh) & 255u], 1u);
        __syncthreads();
        if (warp == 0) {
            uint32_t c8 = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) c8 += hist[lane * 8 + e];
            uint32_t incl = c8;
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= (uint32_t)off) incl += o;
            }
            const uint32_t excl = incl - c8;
            if (excl < want && want <= incl) {
                uint32_t cum = excl, dg = lane * 8;
                for (int e = 0; e < 8; ++e) {
                    if (cum + hist[lane * 8 + e] >= want) { dg = lane * 8 + e; break; }
                    cum += hist[lane * 8 + e];
                }
                red_u[0] = dg;
                red_u[1] = cum;
            }
        }
        __syncthreads();
        prefix |= red_u[0] << sh;
        want -= red_u[1];
        __syncthreads();
    }
    // threads (groups) hold fewer than np values when ngroups * 3 < np: no bound
    const float T = np > nkept ? __int_as_float(0x7f800000) : cr_unord(prefix | 0xFFFFu);
    const float qnorm = sqrtf(qn);
    // + K5t's index packing: the low 7 mantissa bits of a' are replaced, |a'| <= |c|^2 + 2 |q| |c|
    const float E = 4.2e-3f * qnorm * cmax + (float)dim * 4e-7f * (qn + cmax * cmax + 2.0f * qnorm * cmax) + 1e-6f +
                    1.7e-5f * (cmax * cmax + 2.0f * qnorm * cmax);
    const float bound = T + 2.0f * E;
    if (!(m3 > bound)) {  // every cell of this thread's groups is a candidate
        for (uint32_t g = tid; g < ngroups; g += CR_THREADS)
            for (uint32_t c = g * CT_GROUP; c < min(nlist, (g + 1) * CT_GROUP); ++c) cand[atomicAdd(&ncand_s, 1u)] = c;
    } else {
        if (!(m1 > bound) && i1 < nlist) cand[atomicAdd(&ncand_s, 1u)] = i1;
        if (!(m2 > bound) && i2 < nlist) cand[atomicAdd(&ncand_s, 1u)] = i2;
    }
    __syncthreads();
    const uint32_t ncand = ncand_s;
    // exact sq_l2 (distances.cpp:10-17, fp32 in dimension order) of the candidates, chunk by
    // chunk, merged into the running top-np
    uint32_t ntop = 0;
    for (uint32_t c0 = 0; c0 < ncand; c0 += CR_CHUNK) {
        const uint32_t cnk = min((uint32_t)CR_CHUNK, ncand - c0);
        for (uint32_t i = tid; i < cnk; i += CR_THREADS) {
            const uint32_t cell = cand[c0 + i];
            const float* crow = cent + (size_t)cell * dim;
            float acc = 0.0f;
            for (uint32_t d0 = 0; d0 < dim; d0 += 32) {  // dim % 32 == 0 (16 * m, m in {8, 16})
                float4 c4[8];
#pragma unroll
                for (int v = 0; v < 8; ++v) c4[v] = __ldg(reinterpret_cast<const float4*>(crow + d0) + v);
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    const float cv[4] = {c4[v].x, c4[v].y, c4[v].z, c4[v].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float t = __fsub_rn(qs[d0 + 4 * v + e], cv[e]);
                        acc = __fadd_rn(acc, __fmul_rn(t, t));
                    }
                }
            }
            buf[ntop + i] = ((unsigned long long)__float_as_uint(acc) << 32) | cell;
        }
        const uint32_t n = ntop + cnk;
        __syncthreads();
        if (n <= CR_RANKMAX) {  // rank by counting (keys distinct: the low word is the cell)
            unsigned long long* out = buf + CR_BUF / 2;
            for (uint32_t i = tid; i < n; i += CR_THREADS) {
                const unsigned long long ki = buf[i];
                uint32_t rank = 0;
                for (uint32_t j = 0; j < n; ++j) rank += buf[j] < ki;
                if (rank < np) out[rank] = ki;
            }
            __syncthreads();
            for (uint32_t i = tid; i < min(n, np); i += CR_THREADS) buf[i] = out[i];
            __syncthreads();
            ntop = min(n, np);
            continue;
        }
        uint32_t P = 1;
        while (P < n) P <<= 1;
        for (uint32_t i = n + tid; i < P; i += CR_THREADS) buf[i] = ~0ull;
        __syncthreads();
        for (uint32_t size = 2; size <= P; size <<= 1)
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = tid; i < P / 2; i += CR_THREADS) {
                    const uint32_t pos = 2 * i - (i & (stride - 1));
                    const bool asc = (pos & size) == 0;
                    const unsigned long long x = buf[pos], y = buf[pos + stride];
                    if ((x > y) == asc) { buf[pos] = y; buf[pos + stride] = x; }
                }
                __syncthreads();
            }
        ntop = min(n, np);
    }
    for (uint32_t i = tid; i < np; i += CR_THREADS) probe_keys[(size_t)qi * np + i] = i < ntop ? buf[i] : ~0ull;
    if (tid == 0) probe_counts[qi] = ntop;
}

void launch_coarse_rank(const float* q, uint32_t nq, uint32_t dim, const float4* grp, uint32_t nlist, float cmax,
                        const float* cent, uint32_t np, uint32_t* scratch, unsigned long long* probe_keys,
                        uint32_t* probe_counts, cudaStream_t s) {
    if (nq == 0) return;
    const size_t smem = (size_t)CR_BUF * 8 + (size_t)dim * 4;
    set_max_smem((const void*)coarse_rank_kernel, smem);
    coarse_rank_kernel<<<nq, CR_THREADS, smem, s>>>(q, nq, dim, grp, 2 * coarse_tc_tiles(nlist), cmax, cent, nlist,
                                                    np, scratch, probe_keys, probe_counts);
    count_launch();
}

}  // namespace pb
