// kernels_topk.cu -- K3: exact per-query top-k over 64-bit candidate keys.
//
// Implements the SPEC top-k contract: the k
// lexicographically smallest (score, id) pairs, ascending, fewer when fewer
// candidates exist.  It replaces TopK::sorted (flat_index.hpp:81-85), whose
// heap is inverted in the reference.  Keys are
// (fp32 score bits << 32 | 32-bit id rank); scores are >= 0, so unsigned key
// order == (score, id) order and ties resolve to the lower id.
//
// One CTA per query.  <= 2048 candidates: bitonic sort in shared memory.
// More: a 3-pass bucket select -- key range (min, max), a 2048-bucket histogram
// over the bits just below the highest bit where min and max differ, then the
// keys of the buckets up to the k-th one are gathered (usually ~k) and sorted.
// Fallbacks when that set exceeds TK_SEL_KEYS: bitonic sort of all keys (<= 8192,
// in shared memory) or an 8-pass radix select of the k-th key streamed from L2.
// The same kernel merges the per-GPU lists of the multi-GPU path (parts > 1).
#include "poly_b200.cuh"

namespace pb {

constexpr int TK_THREADS = 512;
constexpr uint32_t TK_SMEM_KEYS = 8192;
constexpr int TK_MAXPARTS = 64;
constexpr uint32_t TK_DIRECT = 2048;  // at most this many: sort them all
constexpr uint32_t TK_SEL_KEYS = 2048;  // with 2048 buckets: 88 KB of smem, two CTAs per SM
constexpr uint32_t TK_BUCKETS = 2048;

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
    unsigned long long* sel = sk + TK_SMEM_KEYS;                       // TK_SEL_KEYS
    uint32_t* bh = reinterpret_cast<uint32_t*>(sel + TK_SEL_KEYS);    // TK_BUCKETS
    const bool in_smem = total <= TK_SMEM_KEYS;
    if (in_smem) {  // stage all keys in shared memory
        uint32_t base = 0;
        for (uint32_t p = 0; p < parts; ++p) {
            const unsigned long long* src = cand + p * part_stride + (size_t)q * cap;
            for (uint32_t i = threadIdx.x; i < pc[p]; i += TK_THREADS) sk[base + i] = __ldcg(src + i);
            base += pc[p];
        }
        __syncthreads();
    }
    // key i of the list (shared memory or global)
    auto key_at = [&](uint32_t p, uint32_t i, uint32_t flat) -> unsigned long long {
        return in_smem ? sk[flat] : __ldcg(cand + p * part_stride + (size_t)q * cap + i);
    };
    if (total > TK_DIRECT && kk > 0) {
        // pass 1: key range
        unsigned long long lo = ~0ull, hi = 0;
        {
            uint32_t flat = 0;
            for (uint32_t p = 0; p < parts; ++p) {
                for (uint32_t i = threadIdx.x; i < pc[p]; i += TK_THREADS) {
                    const unsigned long long v = key_at(p, i, flat + i);
                    lo = v < lo ? v : lo;
                    hi = v > hi ? v : hi;
                }
                flat += pc[p];
            }
        }
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, off), b = __shfl_xor_sync(0xffffffffu, hi, off);
            lo = a < lo ? a : lo;
            hi = b > hi ? b : hi;
        }
        __shared__ unsigned long long wlo[TK_THREADS / 32], whi[TK_THREADS / 32];
        if ((threadIdx.x & 31) == 0) { wlo[threadIdx.x >> 5] = lo; whi[threadIdx.x >> 5] = hi; }
        for (uint32_t i = threadIdx.x; i < TK_BUCKETS; i += TK_THREADS) bh[i] = 0;
        __syncthreads();
        lo = ~0ull; hi = 0;
        for (int w = 0; w < TK_THREADS / 32; ++w) {
            lo = wlo[w] < lo ? wlo[w] : lo;
            hi = whi[w] > hi ? whi[w] : hi;
        }
        const unsigned long long span = hi - lo;
        const int top = span ? 63 - __clzll(span) : 0;     // highest differing bit of the range
        constexpr int BB = 31 - __builtin_clz(TK_BUCKETS);  // log2(buckets)
        const int sh = top >= BB ? top - (BB - 1) : 0;      // (span >> sh) < TK_BUCKETS
        // pass 2: histogram
        {
            uint32_t flat = 0;
            for (uint32_t p = 0; p < parts; ++p) {
                for (uint32_t i = threadIdx.x; i < pc[p]; i += TK_THREADS)
                    atomicAdd(&bh[(uint32_t)((key_at(p, i, flat + i) - lo) >> sh)], 1u);
                flat += pc[p];
            }
        }
        __syncthreads();
        // bucket of the kk-th key: per-thread sums of 8 buckets, block scan
        constexpr uint32_t PER = TK_BUCKETS / TK_THREADS;
        uint32_t c = 0;
#pragma unroll
        for (uint32_t j = 0; j < PER; ++j) c += bh[threadIdx.x * PER + j];
        uint32_t incl = c;
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
            if ((threadIdx.x & 31) >= off) incl += o;
        }
        __shared__ uint32_t wsum[TK_THREADS / 32];
        if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = incl;
        __syncthreads();
        uint32_t wbase = 0;
        for (uint32_t w = 0; w < (threadIdx.x >> 5); ++w) wbase += wsum[w];
        incl += wbase;
        const uint32_t excl = incl - c;
        if (excl < kk && kk <= incl) {
            uint32_t cum = excl, b = threadIdx.x * PER;
            for (uint32_t j = 0; j < PER; ++j) {
                cum += bh[b + j];
                if (cum >= kk) { b += j; break; }
            }
            k_s = b;      // bucket holding the kk-th key
            fill_s = cum; // keys in buckets <= b
        }
        __syncthreads();
        const uint32_t nsel = fill_s;
        if (nsel <= TK_SEL_KEYS) {
            // pass 3: gather buckets <= b, sort, emit
            const uint32_t bsel = k_s;
            __syncthreads();
            if (threadIdx.x == 0) fill_s = 0;
            __syncthreads();
            uint32_t flat = 0;
            for (uint32_t p = 0; p < parts; ++p) {
                for (uint32_t i = threadIdx.x; i < pc[p]; i += TK_THREADS) {
                    const unsigned long long v = key_at(p, i, flat + i);
                    if (((v - lo) >> sh) <= bsel) sel[atomicAdd(&fill_s, 1u)] = v;
                }
                flat += pc[p];
            }
            __syncthreads();
            const uint32_t n = fill_s;
            uint32_t P = 1;
            while (P < n) P <<= 1;
            for (uint32_t i = n + threadIdx.x; i < P; i += TK_THREADS) sel[i] = KEY_INF;
            __syncthreads();
            bitonic_sort(sel, P);
            for (uint32_t r = threadIdx.x; r < k; r += TK_THREADS) out[r] = r < kk ? sel[r] : KEY_INF;
            if (threadIdx.x == 0) out_counts[q] = kk;
            return;
        }
        __syncthreads();
    }
    if (in_smem) {
        uint32_t P = 1;
        while (P < total) P <<= 1;
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
    const size_t smem = (TK_SMEM_KEYS + TK_SEL_KEYS) * sizeof(unsigned long long) + TK_BUCKETS * sizeof(uint32_t);
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
