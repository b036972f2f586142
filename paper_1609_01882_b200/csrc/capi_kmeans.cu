// capi_kmeans.cu -- train_coarse's k-means on the GPU ("ivf: one k-means
// codebook of K_coarse centroids over full D"), poly_b200_kmeans in include/poly_b200.h.
//
// Restates the reference's kmeans (proj/src/kmeans.cpp:14-137, KmeansParams kmeans.hpp:10-14):
//   seeding   k-means++ (kmeans.cpp:14-47): the first centroid uniform (Rng::below), then
//             D^2 sampling: target = u01 * sum(min_d2), pick the first point where the
//             running subtraction reaches <= 0; min_d2 = sq_l2 to the nearest chosen
//             centroid (fp32 sq_l2 widened to double).  The min_d2 updates and block sums
//             run on the GPU; the draw itself on the host with the reference's Rng
//             (mt19937_64, u01 = (x >> 11) 2^-53, below = rejection) over the block sums,
//             then the chosen block's values in order.
//   Lloyd     iters x {assign_nearest, objective, per-cell sums in double, centroid =
//             float(sum * (1 / count)), empty cells (ascending) take the farthest member of
//             the currently largest cell} (kmeans.cpp:76-125), then a final assignment.
//             assign_nearest (distances.cpp:56-79) is exact here: K5t/K5q (kernels_coarse.cu)
//             with np = 1 give the nearest cell by fp32 sq_l2 in dimension order, ties to the
//             lower cell (the reference's BLAS GEMM form can flip near-ties; parity of the
//             trained codebook is therefore not bit-exact -- SURVEY.md sec. 8(c), BLAS).
//   n <= k    every point becomes a centroid, cells replicate points cyclically (kmeans.cpp:62-73).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "../../include/poly_b200.h"
#include "host_common.h"
#include "poly_b200.cuh"

using namespace pbh;

namespace pb {

constexpr uint32_t KM_BLOCK = 1024;  // points per D^2 block sum

__device__ __forceinline__ float km_sq_l2(const float* __restrict__ a, const float* __restrict__ b, uint32_t dim) {
    float acc = 0.0f;  // sq_l2 (distances.cpp:10-17): fp32, dimension order, no FMA
    for (uint32_t d = 0; d < dim; ++d) {
        const float t = __fsub_rn(a[d], b[d]);
        acc = __fadd_rn(acc, __fmul_rn(t, t));
    }
    return acc;
}

// min_d2[i] = init ? d2 : min(min_d2[i], d2) with d2 = sq_l2(x_i, c); block sums of min_d2
__global__ void __launch_bounds__(256) km_d2_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim,
                                                    const float* __restrict__ c, int init, double* __restrict__ min_d2,
                                                    double* __restrict__ block_sum) {
    __shared__ double part[8];
    const uint64_t b0 = (uint64_t)blockIdx.x * KM_BLOCK;
    double s = 0.0;
    const uint64_t b1 = n < b0 + KM_BLOCK ? n : b0 + KM_BLOCK;
    for (uint64_t i = b0 + threadIdx.x; i < b1; i += 256) {
        const double d2 = (double)km_sq_l2(x + i * dim, c, dim);
        double v = d2;
        if (!init) {
            const double o = min_d2[i];
            v = d2 < o ? d2 : o;
        }
        min_d2[i] = v;
        s += v;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += part[w];
        block_sum[blockIdx.x] = t;
    }
}

__global__ void km_keys_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim, const float* __restrict__ cent,
                               const uint32_t* __restrict__ assign, unsigned long long* __restrict__ keys) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = assign[i];
        keys[i] = ((unsigned long long)__float_as_uint(km_sq_l2(x + i * dim, cent + (size_t)c * dim, dim)) << 32) | c;
    }
}

__global__ void km_accumulate_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim,
                                     const unsigned long long* __restrict__ keys, double* __restrict__ sums,
                                     unsigned long long* __restrict__ counts, uint32_t* __restrict__ assign,
                                     double* __restrict__ obj) {
    double o = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[i];
        const uint32_t c = (uint32_t)key;
        assign[i] = c;
        o += (double)__uint_as_float((uint32_t)(key >> 32));
        atomicAdd(counts + c, 1ull);
        for (uint32_t d = 0; d < dim; ++d) atomicAdd(sums + (size_t)c * dim + d, (double)x[i * dim + d]);
    }
    for (int s = 16; s > 0; s >>= 1) o += __shfl_down_sync(0xffffffffu, o, s);
    if ((threadIdx.x & 31) == 0) atomicAdd(obj, o);
}

__global__ void km_finalize_kernel(const double* __restrict__ sums, const unsigned long long* __restrict__ counts,
                                   uint32_t k, uint32_t dim, float* __restrict__ cent) {
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (uint64_t)k * dim;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = e / dim;
        if (counts[c] == 0) continue;
        const double inv = 1.0 / (double)counts[c];
        cent[e] = (float)(sums[e] * inv);
    }
}

// farthest member of cell `big` (sq_l2 to its centroid, the first index on ties): per-block
// (d2 bits << 32 | ~index) maxima; the host takes the max of the block results
__global__ void __launch_bounds__(256) km_farthest_kernel(const float* __restrict__ x, uint64_t n, uint32_t dim,
                                                          const uint32_t* __restrict__ assign, uint32_t big,
                                                          const float* __restrict__ cbig,
                                                          unsigned long long* __restrict__ best) {
    unsigned long long m = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (assign[i] != big) continue;
        const float d2 = km_sq_l2(x + i * dim, cbig, dim);
        const unsigned long long key = ((unsigned long long)__float_as_uint(d2) << 32) | (0xFFFFFFFFu - (uint32_t)i);
        m = key > m ? key : m;
    }
    for (int s = 16; s > 0; s >>= 1) {
        const unsigned long long o = __shfl_down_sync(0xffffffffu, m, s);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(best, m);
}

}  // namespace pb

namespace {

// poly::Rng (common.hpp:45-67) over std::mt19937_64
struct RefRng {
    std::mt19937_64 gen;
    explicit RefRng(uint64_t seed) : gen(seed) {}
    double u01() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
    uint64_t below(uint64_t n) {
        if (n <= 1) return 0;
        const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t x;
        do {
            x = gen();
        } while (x >= limit);
        return x % n;
    }
};

struct KmDev {
    float* x = nullptr;
    float* cent = nullptr;
    double* min_d2 = nullptr;
    double* bsum = nullptr;
    double* sums = nullptr;
    unsigned long long* counts = nullptr;
    unsigned long long* keys = nullptr;
    uint32_t* assign = nullptr;
    double* obj = nullptr;
    unsigned long long* best = nullptr;
    float* packed = nullptr;
    float* cnorm = nullptr;
    float4* grp = nullptr;
    uint32_t* rank = nullptr;
    uint32_t* pcount = nullptr;
    ~KmDev() {
        for (void* p : {(void*)x, (void*)cent, (void*)min_d2, (void*)bsum, (void*)sums, (void*)counts, (void*)keys,
                        (void*)assign, (void*)obj, (void*)best, (void*)packed, (void*)cnorm, (void*)grp, (void*)rank,
                        (void*)pcount})
            dfree(p);
    }
};

constexpr uint32_t KM_QB = 2048;  // points per assignment batch

// exact nearest cell of every point: keys[i] = (sq_l2 bits << 32) | cell
void km_assign(KmDev& d, uint64_t n, uint32_t dim, uint32_t k, int num_sms, cudaStream_t s) {
    const bool tc = dim % 32 == 0;
    if (!tc) {  // plain exact kernel (any dim): assign only, distances recomputed below
        pb::launch_assign(d.x, n, dim, d.cent, k, d.assign, s);
        return;
    }
    pb::launch_coarse_pack(d.cent, k, dim, d.packed, d.cnorm, s);
    std::vector<float> hc((size_t)k * dim);
    CK(cudaMemcpyAsync(hc.data(), d.cent, hc.size() * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double cm = 0.0;
    for (uint32_t c = 0; c < k; ++c) {
        double a = 0.0;
        for (uint32_t j = 0; j < dim; ++j) a += (double)hc[(size_t)c * dim + j] * hc[(size_t)c * dim + j];
        cm = std::max(cm, a);
    }
    const float cmax = (float)(std::sqrt(cm) * (1.0 + 1e-5)) + 1e-30f;
    for (uint64_t b0 = 0; b0 < n; b0 += KM_QB) {
        const uint32_t nb = (uint32_t)std::min<uint64_t>(KM_QB, n - b0);
        pb::launch_coarse_tc(d.x + b0 * dim, nb, dim, d.packed, d.cnorm, k, num_sms, d.grp, s);
        pb::launch_coarse_rank(d.x + b0 * dim, nb, dim, d.grp, k, cmax, d.cent, 1, d.rank, d.keys + b0, d.pcount, s);
    }
}

}  // namespace

extern "C" {

int poly_b200_kmeans(const float* x, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed, int device,
                     float* centroids, uint32_t* assign, double* iteration_mse, double* mse) {
    return guard([&] {
        require(n > 0, POLY_B200_INVALID_ARGUMENT, "kmeans on empty data");
        require(k > 0, POLY_B200_INVALID_ARGUMENT, "kmeans with k=0");
        require(x && centroids && dim > 0, POLY_B200_INVALID_ARGUMENT, "null arguments");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, POLY_B200_INVALID_ARGUMENT, "no such CUDA device");
        for (uint64_t i = 0; i < n * dim; ++i)
            require(std::isfinite(x[i]), POLY_B200_INVALID_ARGUMENT, "non-finite entry in vector set");
        DeviceGuard dg(device);
        if (n <= k) {  // kmeans.cpp:62-73
            for (uint32_t c = 0; c < k; ++c) std::memcpy(centroids + (size_t)c * dim, x + (c % n) * dim, dim * 4);
            if (assign)
                for (uint64_t i = 0; i < n; ++i) assign[i] = (uint32_t)i;
            if (mse) *mse = 0.0;
            return;
        }
        int num_sms = 148;
        CK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device));
        cudaStream_t s = nullptr;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{s};
        KmDev d;
        const uint64_t nblk = (n + pb::KM_BLOCK - 1) / pb::KM_BLOCK;
        d.x = dalloc<float>(n * dim);
        d.cent = dalloc<float>((size_t)k * dim);
        d.min_d2 = dalloc<double>(n);
        d.bsum = dalloc<double>(nblk);
        d.sums = dalloc<double>((size_t)k * dim);
        d.counts = dalloc<unsigned long long>(k);
        d.keys = dalloc<unsigned long long>(n);
        d.assign = dalloc<uint32_t>(n);
        d.obj = dalloc<double>(1);
        d.best = dalloc<unsigned long long>(1);
        if (dim % 32 == 0) {
            const size_t npad = (size_t)pb::coarse_tc_tiles(k) * 256;
            d.packed = dalloc<float>(npad * dim);
            d.cnorm = dalloc<float>(npad);
            d.grp = dalloc<float4>((size_t)KM_QB * 2 * pb::coarse_tc_tiles(k));
            d.rank = dalloc<uint32_t>((size_t)KM_QB * k);
            d.pcount = dalloc<uint32_t>(KM_QB);
        }
        CK(cudaMemcpyAsync(d.x, x, n * dim * 4, cudaMemcpyHostToDevice, s));

        // ---- k-means++ seeding (kmeans.cpp:14-47)
        RefRng rng(seed);
        const uint64_t first = rng.below(n);
        CK(cudaMemcpyAsync(d.cent, d.x + first * dim, dim * 4, cudaMemcpyDeviceToDevice, s));
        std::vector<double> bs(nblk), blk(pb::KM_BLOCK);
        for (uint32_t c = 0; c < k; ++c) {
            if (c > 0) {
                double total = 0.0;
                for (double v : bs) total += v;
                uint64_t pick = n - 1;
                if (total <= 0.0) {
                    pick = rng.below(n);
                } else {
                    double target = rng.u01() * total;
                    uint64_t b = 0;
                    for (; b + 1 < nblk && target - bs[b] > 0.0; ++b) target -= bs[b];
                    const uint64_t i0 = b * pb::KM_BLOCK, cnt = std::min<uint64_t>(pb::KM_BLOCK, n - i0);
                    CK(cudaMemcpyAsync(blk.data(), d.min_d2 + i0, cnt * 8, cudaMemcpyDeviceToHost, s));
                    CK(cudaStreamSynchronize(s));
                    for (uint64_t i = 0; i < cnt; ++i) {
                        target -= blk[i];
                        if (target <= 0.0) {
                            pick = i0 + i;
                            break;
                        }
                    }
                }
                CK(cudaMemcpyAsync(d.cent + (size_t)c * dim, d.x + pick * dim, dim * 4, cudaMemcpyDeviceToDevice, s));
            }
            pb::km_d2_kernel<<<(unsigned)nblk, 256, 0, s>>>(d.x, n, dim, d.cent + (size_t)c * dim, c == 0, d.min_d2,
                                                            d.bsum);
            pb::count_launch();
            if (c + 1 < k) {
                CK(cudaMemcpyAsync(bs.data(), d.bsum, nblk * 8, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
            }
        }

        // ---- Lloyd iterations (kmeans.cpp:76-125)
        std::vector<unsigned long long> cnt(k);
        auto assign_and_objective = [&](double* out_mse) {
            km_assign(d, n, dim, k, num_sms, s);
            if (dim % 32 != 0) {  // keys for the objective from the exact assignment
                pb::km_keys_kernel<<<num_sms * 4, 256, 0, s>>>(d.x, n, dim, d.cent, d.assign, d.keys);
                pb::count_launch();
            }
            CK(cudaMemsetAsync(d.sums, 0, (size_t)k * dim * 8, s));
            CK(cudaMemsetAsync(d.counts, 0, (size_t)k * 8, s));
            CK(cudaMemsetAsync(d.obj, 0, 8, s));
            pb::km_accumulate_kernel<<<num_sms * 8, 256, 0, s>>>(d.x, n, dim, d.keys, d.sums, d.counts, d.assign, d.obj);
            pb::count_launch();
            double obj = 0.0;
            CK(cudaMemcpyAsync(&obj, d.obj, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            CK(cudaGetLastError());
            *out_mse = obj / (double)n;
        };
        for (uint32_t it = 0; it < iters; ++it) {
            double m = 0.0;
            assign_and_objective(&m);
            if (iteration_mse) iteration_mse[it] = m;
            pb::km_finalize_kernel<<<num_sms * 4, 256, 0, s>>>(d.sums, d.counts, k, dim, d.cent);
            pb::count_launch();
            CK(cudaMemcpyAsync(cnt.data(), d.counts, (size_t)k * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            // empty cells: the farthest member of the currently largest cell, ascending cells
            for (uint32_t c = 0; c < k; ++c) {
                if (cnt[c] != 0) continue;
                uint32_t big = 0;
                for (uint32_t o = 1; o < k; ++o)
                    if (cnt[o] > cnt[big]) big = o;
                if (cnt[big] == 0) break;
                CK(cudaMemsetAsync(d.best, 0, 8, s));
                pb::km_farthest_kernel<<<num_sms * 4, 256, 0, s>>>(d.x, n, dim, d.assign, big,
                                                                   d.cent + (size_t)big * dim, d.best);
                pb::count_launch();
                unsigned long long best = 0;
                CK(cudaMemcpyAsync(&best, d.best, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                const uint64_t far = 0xFFFFFFFFu - (uint32_t)best;
                CK(cudaMemcpyAsync(d.cent + (size_t)c * dim, d.x + far * dim, dim * 4, cudaMemcpyDeviceToDevice, s));
                CK(cudaMemcpyAsync(d.assign + far, &c, 4, cudaMemcpyHostToDevice, s));
                CK(cudaStreamSynchronize(s));
                cnt[c] = 1;
                --cnt[big];
            }
        }
        double m = 0.0;
        assign_and_objective(&m);
        if (mse) *mse = m;
        CK(cudaMemcpyAsync(centroids, d.cent, (size_t)k * dim * 4, cudaMemcpyDeviceToHost, s));
        if (assign) CK(cudaMemcpyAsync(assign, d.assign, n * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
