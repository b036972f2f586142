// kernels_encode.cu -- K1 (LUT + query code) and K0 (database encoder).
//
// Both restate the reference's fp32 arithmetic bit for bit:
//   sq_l2          distances.cpp:10-17   acc = 0; d = a - b; acc += d * d   (t order)
//   compute_lut    pq.cpp:91-105         LUT[sq][j] = sq_l2(q_sq, c_{sq,j})
//   permuted_lut   pq.cpp:107-119        LUTp[sq][perm[sq][j]] = LUT[sq][j]
//   encode         pq.cpp:29-45          argmin_j with strict <, store perm[sq][best]
// using __fsub_rn/__fmul_rn/__fadd_rn so nvcc cannot contract to FFMA.
#include "poly_b200.cuh"
#include "synth.cuh"

namespace pb {

__device__ __forceinline__ float sq_l2_16(const float* a, const float4* c) {
    float acc = 0.0f;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        const float4 cc = c[v];
        float d;
        d = __fsub_rn(a[4 * v + 0], cc.x); acc = __fadd_rn(acc, __fmul_rn(d, d));
        d = __fsub_rn(a[4 * v + 1], cc.y); acc = __fadd_rn(acc, __fmul_rn(d, d));
        d = __fsub_rn(a[4 * v + 2], cc.z); acc = __fadd_rn(acc, __fmul_rn(d, d));
        d = __fsub_rn(a[4 * v + 3], cc.w); acc = __fadd_rn(acc, __fmul_rn(d, d));
    }
    return acc;
}

// ------------------------------------------------------------------ K1
// grid (nq, m), 256 threads: thread j owns centroid j of sub-quantizer blockIdx.y.
__global__ void __launch_bounds__(256) lut_kernel(const float* __restrict__ queries, uint32_t dim, uint32_t m,
                                                  const float* __restrict__ codebooks,
                                                  const uint16_t* __restrict__ perms, float* __restrict__ lutp,
                                                  uint8_t* __restrict__ qcodes) {
    const uint32_t qi = blockIdx.x, sq = blockIdx.y, j = threadIdx.x;
    __shared__ float sub[DSUB];
    __shared__ float wv[8];
    __shared__ uint32_t wj[8];
    if (j < DSUB) sub[j] = queries[(size_t)qi * dim + sq * DSUB + j];
    __syncthreads();
    float a[DSUB];
#pragma unroll
    for (int t = 0; t < DSUB; ++t) a[t] = sub[t];
    const float d = sq_l2_16(a, reinterpret_cast<const float4*>(codebooks + ((size_t)sq * KSUB + j) * DSUB));
    const uint32_t p = perms[sq * KSUB + j];
    lutp[((size_t)qi * m + sq) * KSUB + p] = d;
    // argmin over j, ties -> lowest j (== the strict-< sequential scan)
    float bv = d;
    uint32_t bj = j;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_down_sync(0xffffffffu, bv, off);
        const uint32_t oj = __shfl_down_sync(0xffffffffu, bj, off);
        if (ov < bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
    }
    if ((j & 31) == 0) { wv[j >> 5] = bv; wj[j >> 5] = bj; }
    __syncthreads();
    if (j == 0) {
        for (int w = 1; w < 8; ++w)
            if (wv[w] < bv || (wv[w] == bv && wj[w] < bj)) { bv = wv[w]; bj = wj[w]; }
        qcodes[(size_t)qi * m + sq] = static_cast<uint8_t>(perms[sq * KSUB + bj]);
    }
}

void launch_lut(const float* queries, uint32_t nq, uint32_t dim, uint32_t m, const float* codebooks,
                const uint16_t* perms, float* lutp, uint8_t* qcodes, cudaStream_t s) {
    if (nq == 0) return;
    lut_kernel<<<dim3(nq, m), 256, 0, s>>>(queries, dim, m, codebooks, perms, lutp, qcodes);
    count_launch();
}

// ------------------------------------------------------------------ K0
// One thread per vector; the codebook of sub-quantizer sq is staged in shared
// memory (16 KB) and read with broadcast loads.
constexpr int ENC_THREADS = 128;

template <bool SYNTH>
__global__ void __launch_bounds__(ENC_THREADS) encode_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim,
                                                             uint32_t m, const float* __restrict__ codebooks,
                                                             const uint16_t* __restrict__ perms,
                                                             uint8_t* __restrict__ codes, uint64_t seed,
                                                             uint32_t stream_id, uint64_t row0,
                                                             const float* __restrict__ centers, uint32_t ncent,
                                                             int normalize) {
    __shared__ float4 cb[KSUB * DSUB / 4];
    const uint64_t i = (uint64_t)blockIdx.x * ENC_THREADS + threadIdx.x;
    const bool live = i < n;
    uint64_t key = 0;
    const float* crow = nullptr;
    float inv = 1.0f;
    if (SYNTH && live) {
        key = row_key(seed, stream_id, row0 + i);
        crow = centers + (size_t)synth_center(key, ncent) * dim;
        if (normalize) inv = synth_inv_norm(crow, key, dim);
    }
    for (uint32_t sq = 0; sq < m; ++sq) {
        __syncthreads();
        const float4* src = reinterpret_cast<const float4*>(codebooks + (size_t)sq * KSUB * DSUB);
        for (int e = threadIdx.x; e < KSUB * DSUB / 4; e += ENC_THREADS) cb[e] = src[e];
        __syncthreads();
        if (!live) continue;
        float a[DSUB];
        if (SYNTH) {
#pragma unroll
            for (int t = 0; t < DSUB; ++t) {
                const float v = synth_coord(crow, key, sq * DSUB + t);
                a[t] = normalize ? __fmul_rn(v, inv) : v;
            }
        } else {
            const float4* xr = reinterpret_cast<const float4*>(x + i * dim + sq * DSUB);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const float4 f = xr[v];
                a[4 * v] = f.x; a[4 * v + 1] = f.y; a[4 * v + 2] = f.z; a[4 * v + 3] = f.w;
            }
        }
        uint32_t best = 0;
        float best_d = sq_l2_16(a, cb);
        for (uint32_t j = 1; j < KSUB; ++j) {
            const float d = sq_l2_16(a, cb + j * (DSUB / 4));
            if (d < best_d) { best_d = d; best = j; }   // pq.cpp:38 ties keep the lowest index
        }
        codes[i * m + sq] = static_cast<uint8_t>(perms[sq * KSUB + best]);
    }
}

void launch_encode(const float* x, uint64_t n, uint32_t dim, uint32_t m, const float* codebooks,
                   const uint16_t* perms, uint8_t* codes, cudaStream_t s) {
    if (n == 0) return;
    const uint64_t blocks = (n + ENC_THREADS - 1) / ENC_THREADS;
    encode_kernel<false><<<(unsigned)blocks, ENC_THREADS, 0, s>>>(x, n, dim, m, codebooks, perms, codes, 0, 0, 0,
                                                                  nullptr, 0, 0);
    count_launch();
}

void launch_synth_encode(uint64_t seed, uint32_t stream_id, uint64_t row0, uint64_t n, const float* centers,
                         uint32_t ncent, uint32_t dim, int normalize, uint32_t m, const float* codebooks,
                         const uint16_t* perms, uint8_t* codes, cudaStream_t s) {
    if (n == 0) return;
    const uint64_t blocks = (n + ENC_THREADS - 1) / ENC_THREADS;
    encode_kernel<true><<<(unsigned)blocks, ENC_THREADS, 0, s>>>(nullptr, n, dim, m, codebooks, perms, codes, seed,
                                                                 stream_id, row0, centers, ncent, normalize);
    count_launch();
}

// ------------------------------------------------------------------ generator (tests)
__global__ void gen_points_kernel(uint64_t seed, uint32_t stream_id, uint64_t row0, uint64_t n,
                                  const float* __restrict__ centers, uint32_t ncent, uint32_t dim, int normalize,
                                  float* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t key = row_key(seed, stream_id, row0 + i);
    const float* crow = centers + (size_t)synth_center(key, ncent) * dim;
    const float inv = normalize ? synth_inv_norm(crow, key, dim) : 1.0f;
    for (uint32_t t = 0; t < dim; ++t) {
        const float v = synth_coord(crow, key, t);
        out[i * dim + t] = normalize ? __fmul_rn(v, inv) : v;
    }
}

void launch_gen_points(uint64_t seed, uint32_t stream_id, uint64_t row0, uint64_t n, const float* centers,
                       uint32_t ncent, uint32_t dim, int normalize, float* out, cudaStream_t s) {
    if (n == 0) return;
    gen_points_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(seed, stream_id, row0, n, centers, ncent, dim,
                                                                   normalize, out);
    count_launch();
}

// ------------------------------------------------------------------ calibration / relabel
// hist[q][h] += #codes at Hamming distance h (flat_index.hpp:128-132 needs the
// survivor fraction for every tau).  One CTA per (query, code slab).
__global__ void hamming_hist_kernel(const uint8_t* __restrict__ codes, uint64_t n, uint32_t cb,
                                    const uint8_t* __restrict__ qcodes, unsigned long long* __restrict__ hist) {
    __shared__ uint32_t h[129];
    const uint32_t q = blockIdx.y;
    for (int i = threadIdx.x; i < 129; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t words = cb / 8;
    uint64_t qw[2] = {0, 0};
    for (uint32_t w = 0; w < words; ++w) qw[w] = reinterpret_cast<const uint64_t*>(qcodes + (size_t)q * cb)[w];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t d = 0;
        for (uint32_t w = 0; w < words; ++w) d += __popcll(reinterpret_cast<const uint64_t*>(codes + i * cb)[w] ^ qw[w]);
        atomicAdd(&h[d], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= (int)(cb * 8); i += blockDim.x)
        if (h[i]) atomicAdd(&hist[(size_t)q * (cb * 8 + 1) + i], (unsigned long long)h[i]);
}

void launch_hamming_hist(const uint8_t* codes, uint64_t n, uint32_t cb, const uint8_t* qcodes, uint32_t nq,
                         unsigned long long* hist, cudaStream_t s) {
    if (n == 0 || nq == 0) return;
    const unsigned slabs = (unsigned)((n + 256 * 64 - 1) / (256 * 64));
    hamming_hist_kernel<<<dim3(slabs < 148 ? slabs : 148, nq), 256, 0, s>>>(codes, n, cb, qcodes, hist);
    count_launch();
}

__global__ void relabel_kernel(uint8_t* __restrict__ codes, uint64_t total, uint32_t m,
                               const uint8_t* __restrict__ maps) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
        codes[i] = maps[(i % m) * KSUB + codes[i]];
}

void launch_relabel(uint8_t* codes, uint64_t n, uint32_t m, const uint8_t* maps, cudaStream_t s) {
    if (n == 0) return;
    relabel_kernel<<<148 * 8, 256, 0, s>>>(codes, n * m, m, maps);
    count_launch();
}

}  // namespace pb
