// kernels_topk.cu -- K3: exact per-query top-k over 64-bit candidate keys.
//
// Implements the SPEC top-k contract: the k
// lexicographically smallest (score, id) pairs, ascending, fewer when fewer
// candidates exist.  It replaces TopK::sorted (flat_index.hpp:81-85), whose
// heap is inverted in the reference.  Keys are
// (fp32 score bits << 32 | 32-bit id rank); scores are >= 0, so unsigned key
// order == (score, id) order and ties resolve to the lower id.
//
// One CTA per query.  <= 8192 candidates: bitonic sort in shared memory.
// More: 8-pass radix select of the k-th key streamed from L2, then the k keys
// <= it are gathered and sorted.  The same kernel merges the per-GPU lists of
// the multi-GPU path (parts > 1).
#include "poly_b200.cuh"

namespace pb {

constexpr int TK_THREADS = 512;
constexpr uint32_t TK_SMEM_KEYS = 8192;
constexpr int TK_MAXPARTS = 64;

__device__ __forceinline__ void bitonic_sort(unsigned long long* s, uint32_t p) {
    for (uint32_t size = 2; size <= p; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < p / 2; i += TK_THREADS) {
                const uint32_t pos = 2 * i - (i & (stride - 1));
                const bool asc = (pos & size) == 0;
                const unsigned long long x = s[pos], y = s[pos + stride];
                if ((x > y) == asc) { s[pos] = y; s[pos + stride] = x; }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(TK_THREADS) topk_kernel(const unsigned long long* __restrict__ cand,
                                                          const uint32_t* __restrict__ ccount, uint32_t cap,
                                                          uint32_t parts, uint64_t part_stride, uint64_t count_stride,
                                                          uint32_t nq, uint32_t k,
                                                          unsigned long long* __restrict__ out_keys,
                                                          uint32_t* __restrict__ out_counts) {
    extern __shared__ unsigned long long sk[];
    __shared__ uint32_t pc[TK_MAXPARTS];
    __shared__ uint32_t hist[256];
    __shared__ unsigned long long prefix_s;
    __shared__ uint32_t k_s, fill_s;
    const uint32_t q = blockIdx.x;
    if (threadIdx.x < parts) pc[threadIdx.x] = min(ccount[(size_t)threadIdx.x * count_stride + q], cap);
    __syncthreads();
    uint32_t total = 0;
    for (uint32_t p = 0; p < parts; ++p) total += pc[p];
    const uint32_t kk = min(k, total);
    unsigned long long* out = out_keys + (size_t)q * k;
    if (total <= TK_SMEM_KEYS) {
        uint32_t P = 1;
        while (P < total) P <<= 1;
        uint32_t base = 0;
        for (uint32_t p = 0; p < parts; ++p) {
            const unsigned long long* src = cand + p * part_stride + (size_t)q * cap;
            for (uint32_t i = threadIdx.x; i < pc[p]; i += TK_THREADS) sk[base + i] = __ldcg(src + i);
            base += pc[p];
        }
        for (uint32_t i = total + threadIdx.x; i < P; i += TK_THREADS) sk[i] = KEY_INF;
        __syncthreads();
        bitonic_sort(sk, P);
    } else {
        // radix select of the kk-th smallest key over all parts
        unsigned long long prefix = 0, mask = 0;
        uint32_t want = kk;
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int i = threadIdx.x; i < 256; i += TK_THREADS) hist[i] = 0;
            __syncthreads();
            for (uint32_t p = 0; p < parts; ++p) {
                const unsigned long long* src = cand + p * part_stride + (size_t)q * cap;
                for (uint32_t i = threadIdx.x; i < pc[p]; i += TK_THREADS) {
                    const unsigned long long v = __ldcg(src + i);
                    if ((v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 0xFFu], 1u);
                }
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                const int lane = threadIdx.x;
                uint32_t c[8], s = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) { c[j] = hist[lane * 8 + j]; s += c[j]; }
                uint32_t incl = s;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += o;
                }
                const uint32_t excl = incl - s;
                if (excl < want && want <= incl) {
                    uint32_t r = want - excl;
                    int digit = lane * 8 + 7;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        if (r <= c[j]) { digit = lane * 8 + j; break; }
                        r -= c[j];
                    }
                    prefix_s = prefix | ((unsigned long long)digit << shift);
                    k_s = r;
                }
            }
            __syncthreads();
            prefix = prefix_s;
            want = k_s;
            mask |= 0xFFull << shift;
        }
        // gather the kk keys <= kth (keys are distinct)
        if (threadIdx.x == 0) fill_s = 0;
        __syncthreads();
        for (uint32_t p = 0; p < parts; ++p) {
            const unsigned long long* src = cand + p * part_stride + (size_t)q * cap;
            for (uint32_t i = threadIdx.x; i < pc[p]; i += TK_THREADS) {
                const unsigned long long v = __ldcg(src + i);
                if (v <= prefix) sk[atomicAdd(&fill_s, 1u)] = v;
            }
        }
        uint32_t P = 1;
        while (P < kk) P <<= 1;
        __syncthreads();
        for (uint32_t i = kk + threadIdx.x; i < P; i += TK_THREADS) sk[i] = KEY_INF;
        __syncthreads();
        bitonic_sort(sk, P);
    }
    for (uint32_t r = threadIdx.x; r < k; r += TK_THREADS) out[r] = r < kk ? sk[r] : KEY_INF;
    if (threadIdx.x == 0) out_counts[q] = kk;
}

void launch_topk(const unsigned long long* cand, const uint32_t* ccount, uint32_t cap, uint32_t parts,
                 uint64_t part_stride, uint64_t count_stride, uint32_t nq, uint32_t k, unsigned long long* out_keys,
                 uint32_t* out_counts, cudaStream_t s) {
    if (nq == 0 || k == 0) return;
    const size_t smem = TK_SMEM_KEYS * sizeof(unsigned long long);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    topk_kernel<<<nq, TK_THREADS, smem, s>>>(cand, ccount, cap, parts, part_stride, count_stride, nq, k, out_keys,
                                              out_counts);
    count_launch();
}

// key -> (id, score); unfilled slots get id -1 and score +inf (C-ABI contract).
__global__ void keys_to_ids_kernel(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ counts,
                                   uint32_t nq, uint32_t k, const int64_t* __restrict__ rank_to_id,
                                   int64_t* __restrict__ out_ids, float* __restrict__ out_scores,
                                   uint32_t* __restrict__ out_counts) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (uint64_t)nq * k) return;
    const uint32_t q = (uint32_t)(i / k), r = (uint32_t)(i % k);
    const uint32_t c = counts ? counts[q] : 0;
    if (r < c) {
        const unsigned long long key = keys[i];
        const uint32_t low = (uint32_t)key;
        out_ids[i] = rank_to_id ? rank_to_id[low] : (int64_t)low;
        out_scores[i] = __uint_as_float((uint32_t)(key >> 32));
    } else {
        out_ids[i] = -1;
        out_scores[i] = __int_as_float(0x7f800000);
    }
    if (r == 0 && out_counts) out_counts[q] = c;
}

void launch_keys_to_ids(const unsigned long long* keys, const uint32_t* counts, uint32_t nq, uint32_t k,
                        const int64_t* rank_to_id, int64_t* out_ids, float* out_scores, uint32_t* out_counts,
                        cudaStream_t s) {
    const uint64_t total = (uint64_t)nq * k;
    if (total == 0) return;
    keys_to_ids_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(keys, counts, nq, k, rank_to_id, out_ids,
                                                                        out_scores, out_counts);
    count_launch();
}

}  // namespace pb

namespace pb {
__global__ void or_flag_kernel(uint32_t* dst, const uint32_t* src) { *dst |= *src; }
void launch_or_flag(uint32_t* dst, const uint32_t* src, cudaStream_t s) {
    or_flag_kernel<<<1, 1, 0, s>>>(dst, src);
    count_launch();
}
}  // namespace pb

namespace pb {
// thr[q] = min(thr[q], k-th key of the warm-up sample + 1) -- +1 so that key
// itself is appended again by the full scan; unchanged when the sample held
// fewer than k candidates.
__global__ void seed_thr_kernel(const unsigned long long* keys, const uint32_t* counts, uint32_t nq, uint32_t k,
                                unsigned long long* thr) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < nq && counts[q] >= k) {
        const unsigned long long t = keys[(size_t)q * k + k - 1] + 1;
        if (t < thr[q]) thr[q] = t;
    }
}
void launch_seed_thr(const unsigned long long* keys, const uint32_t* counts, uint32_t nq, uint32_t k,
                     unsigned long long* thr, cudaStream_t s) {
    seed_thr_kernel<<<(nq + 127) / 128, 128, 0, s>>>(keys, counts, nq, k, thr);
    count_launch();
}
}  // namespace pb
