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
// More: an iterative bucket select -- key range (min, max), then 2048-bucket
// histograms that narrow to the bucket of the k-th key (11 bits per pass) until
// the keys at or below it fit the select buffer (typically one pass; duplicate
// scores need more), then a bitonic sort of those.  Keys come from shared memory
// (<= 8192 candidates) or L2.  The same kernel merges the per-GPU lists of the
// multi-GPU path (parts > 1).
#include "poly_b200.cuh"

namespace pb {

constexpr int TK_THREADS = 512;
constexpr int TK_MAXPARTS = 64;
#ifndef POLY_TK_DIRECT
#define POLY_TK_DIRECT 512  // IVF A/B: 2048 -> 512 cut the K3 rounds ~6% (flat path: no effect)
#endif
constexpr uint32_t TK_DIRECT = POLY_TK_DIRECT;  // at most this many: sort them all
constexpr uint32_t TK_BUCKETS = 2048;
#ifndef POLY_TK_RANK
#define POLY_TK_RANK 128
#endif
constexpr uint32_t TK_RANK = POLY_TK_RANK;  // at most this many keys to order: rank by counting
#ifndef POLY_TK_SMALLK_KEYS  // keys staged in shared memory when k <= 512
#define POLY_TK_SMALLK_KEYS 6144  // A/B on config 2 (10,000-query steps): 4096 8.61, 6144 8.37, 8192 8.52 ms; config 1 flat
#endif

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

// SMEM_KEYS: keys staged in shared memory (more come from L2); SEL_KEYS: the select
// buffer (>= k + 1).  Two configurations: 8192 / 4096 (104 KB, two CTAs per SM) for
// any k <= 2048, and POLY_TK_SMALLK_KEYS (6144) / 1024 (65 KB, three CTAs per SM) for k <= 512.
template <uint32_t TK_SMEM_KEYS, uint32_t TK_SEL_KEYS>
__global__ void __launch_bounds__(TK_THREADS) topk_kernel(const unsigned long long* __restrict__ cand,
                                                          const uint32_t* __restrict__ ccount, uint32_t cap,
                                                          uint32_t parts, uint64_t part_stride, uint64_t count_stride,
                                                          uint32_t nq, uint32_t k,
                                                          unsigned long long* __restrict__ out_keys,
                                                          uint32_t* __restrict__ out_counts) {
    extern __shared__ unsigned long long sk[];
    __shared__ uint32_t pc[TK_MAXPARTS];
    __shared__ unsigned long long wlo[TK_THREADS / 32], whi[TK_THREADS / 32];
    __shared__ uint32_t wsum[TK_THREADS / 32];
    __shared__ uint32_t b_s, below_s, inb_s, fill_s;
    const uint32_t q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < parts) pc[tid] = min(ccount[(size_t)tid * count_stride + q], cap);
    __syncthreads();
    uint32_t total = 0;
    for (uint32_t p = 0; p < parts; ++p) total += pc[p];
    const uint32_t kk = min(k, total);
    unsigned long long* out = out_keys + (size_t)q * k;
    unsigned long long* sel = sk + TK_SMEM_KEYS;                      // TK_SEL_KEYS
    uint32_t* bh = reinterpret_cast<uint32_t*>(sel + TK_SEL_KEYS);   // TK_BUCKETS
    const bool in_smem = total <= TK_SMEM_KEYS;
    if (in_smem) {  // stage all keys in shared memory
        uint32_t base = 0;
        for (uint32_t p = 0; p < parts; ++p) {
            const unsigned long long* src = cand + p * part_stride + (size_t)q * cap;
            const uint32_t n = pc[p];
            for (uint32_t i0 = tid; i0 < n; i0 += 4 * TK_THREADS) {  // 4 loads in flight
                unsigned long long v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i0 + u * TK_THREADS < n) v[u] = __ldcg(src + i0 + u * TK_THREADS);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i0 + u * TK_THREADS < n) sk[base + i0 + u * TK_THREADS] = v[u];
            }
            base += n;
        }
        __syncthreads();
    }
    // visit every key of the list (shared memory or L2)
    auto for_keys = [&](auto&& f) {
        uint32_t flat = 0;
        for (uint32_t p = 0; p < parts; ++p) {
            const unsigned long long* src = cand + p * part_stride + (size_t)q * cap;
            for (uint32_t i = tid; i < pc[p]; i += TK_THREADS) f(in_smem ? sk[flat + i] : __ldcg(src + i));
            flat += pc[p];
        }
    };
    unsigned long long* srt = sk;  // what gets sorted: all keys (small lists) or the selected ones
    uint32_t n = total;
    if (total > TK_DIRECT && kk > 0) {
        // Iterative bucket select of the kk smallest keys (keys are distinct).  The range
        // [rlo, rlo + (TK_BUCKETS << sh)) holds the kk-th key; keys below it are already
        // known to be among the kk smallest and sit in sel[0, fill).  Each pass histograms
        // the range; the buckets below the kk-th one are kept, and if the kk-th bucket fits
        // too the select ends, else the range narrows to that bucket (11 bits finer).
        unsigned long long lo = ~0ull, hi = 0;
        for_keys([&](unsigned long long v) {
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
        });
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, off), b = __shfl_xor_sync(0xffffffffu, hi, off);
            lo = a < lo ? a : lo;
            hi = b > hi ? b : hi;
        }
        if (lane == 0) { wlo[warp] = lo; whi[warp] = hi; }
        if (tid == 0) fill_s = 0;
        __syncthreads();
        lo = ~0ull; hi = 0;
        for (int w = 0; w < TK_THREADS / 32; ++w) {
            lo = wlo[w] < lo ? wlo[w] : lo;
            hi = whi[w] > hi ? whi[w] : hi;
        }
        constexpr int BB = 31 - __builtin_clz(TK_BUCKETS);  // log2(buckets)
        const unsigned long long span = hi - lo;
        const int top = span ? 63 - __clzll(span) : 0;      // highest differing bit of the range
        int sh = top >= BB ? top - (BB - 1) : 0;            // (span >> sh) < TK_BUCKETS
        unsigned long long rlo = lo;
        uint32_t want = kk;
        for (;;) {
            for (uint32_t i = tid; i < TK_BUCKETS; i += TK_THREADS) bh[i] = 0;
            __syncthreads();
            for_keys([&](unsigned long long v) {
                if (v >= rlo && ((v - rlo) >> sh) < TK_BUCKETS) atomicAdd(&bh[(uint32_t)((v - rlo) >> sh)], 1u);
            });
            __syncthreads();
            // bucket b of the want-th key of the range: per-thread sums, block scan
            constexpr uint32_t PER = TK_BUCKETS / TK_THREADS;
            uint32_t c = 0;
#pragma unroll
            for (uint32_t j = 0; j < PER; ++j) c += bh[tid * PER + j];
            uint32_t incl = c;
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= (uint32_t)off) incl += o;
            }
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            for (uint32_t w = 0; w < warp; ++w) incl += wsum[w];
            const uint32_t excl = incl - c;
            if (excl < want && want <= incl) {
                uint32_t cum = excl, b = tid * PER;
                for (uint32_t j = 0; j < PER; ++j) {
                    if (cum + bh[tid * PER + j] >= want) { b = tid * PER + j; break; }
                    cum += bh[tid * PER + j];
                }
                b_s = b;
                below_s = cum;          // keys of the range in buckets < b
                inb_s = bh[b];          // keys in bucket b
            }
            __syncthreads();
            const uint32_t b = b_s, below = below_s, inb = inb_s, fill = fill_s;
            const bool done = fill + below + inb <= TK_SEL_KEYS;
            const uint32_t last = done ? b : b - 1;  // keep buckets <= last (none when b == 0 and not done)
            __syncthreads();
            if (done || b > 0)
                for_keys([&](unsigned long long v) {
                    if (v >= rlo && ((v - rlo) >> sh) <= last) sel[atomicAdd(&fill_s, 1u)] = v;
                });
            __syncthreads();
            if (done) break;
            rlo += (unsigned long long)b << sh;  // narrow to bucket b
            want -= below;
            sh = sh > BB ? sh - BB : 0;
        }
        srt = sel;
        n = fill_s;
    }
    __syncthreads();
    if (n <= TK_RANK) {
        // rank by counting (2 barriers instead of a bitonic network); ties by position,
        // so the ranks are a permutation even for equal keys
        for (uint32_t i = tid; i < n; i += TK_THREADS) {
            const unsigned long long ki = srt[i];
            uint32_t rank = 0;
            for (uint32_t j = 0; j < n; ++j) {
                const unsigned long long kj = srt[j];
                rank += kj < ki || (kj == ki && j < i);
            }
            if (rank < kk) out[rank] = ki;
        }
        for (uint32_t r = kk + tid; r < k; r += TK_THREADS) out[r] = KEY_INF;
    } else {
        uint32_t P = 1;
        while (P < n) P <<= 1;
        for (uint32_t i = n + tid; i < P; i += TK_THREADS) srt[i] = KEY_INF;
        __syncthreads();
        bitonic_sort(srt, P);
        for (uint32_t r = tid; r < k; r += TK_THREADS) out[r] = r < kk ? srt[r] : KEY_INF;
    }
    if (tid == 0) out_counts[q] = kk;
}

template <uint32_t SK, uint32_t SEL>
static void launch_topk_cfg(const unsigned long long* cand, const uint32_t* ccount, uint32_t cap, uint32_t parts,
                            uint64_t part_stride, uint64_t count_stride, uint32_t nq, uint32_t k,
                            unsigned long long* out_keys, uint32_t* out_counts, cudaStream_t s) {
    const size_t smem = (SK + SEL) * sizeof(unsigned long long) + TK_BUCKETS * sizeof(uint32_t);
    set_max_smem((const void*)topk_kernel<SK, SEL>, smem);
    topk_kernel<SK, SEL><<<nq, TK_THREADS, smem, s>>>(cand, ccount, cap, parts, part_stride, count_stride, nq, k,
                                                      out_keys, out_counts);
}

void launch_topk(const unsigned long long* cand, const uint32_t* ccount, uint32_t cap, uint32_t parts,
                 uint64_t part_stride, uint64_t count_stride, uint32_t nq, uint32_t k, unsigned long long* out_keys,
                 uint32_t* out_counts, cudaStream_t s) {
    if (nq == 0 || k == 0) return;
    if (k <= 512)
        launch_topk_cfg<POLY_TK_SMALLK_KEYS, 1024>(cand, ccount, cap, parts, part_stride, count_stride, nq, k, out_keys,
                                                   out_counts, s);
    else
        launch_topk_cfg<8192, 4096>(cand, ccount, cap, parts, part_stride, count_stride, nq, k, out_keys, out_counts, s);
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
// Between the IVF rounds: thr[q] = k-th key of round 1 + 1 (as seed_thr_kernel),
// and the query's candidate list is cut down to its round-1 top-k, so the final
// K3 ranks k + (round-2 candidates) keys: top-k(A u B) = top-k(top-k(A) u B).
__global__ void seed_compact_kernel(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ counts,
                                    uint32_t k, unsigned long long* __restrict__ thr,
                                    unsigned long long* __restrict__ cand, uint32_t cap,
                                    uint32_t* __restrict__ ccount) {
    const uint32_t q = blockIdx.x, c = counts[q];
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) cand[(size_t)q * cap + i] = keys[(size_t)q * k + i];
    if (threadIdx.x == 0) {
        ccount[q] = c;
        if (c >= k) {
            const unsigned long long t = keys[(size_t)q * k + k - 1] + 1;
            if (t < thr[q]) thr[q] = t;
        }
    }
}
void launch_seed_compact(const unsigned long long* keys, const uint32_t* counts, uint32_t nq, uint32_t k,
                         unsigned long long* thr, unsigned long long* cand, uint32_t cap, uint32_t* ccount,
                         cudaStream_t s) {
    if (nq == 0) return;
    seed_compact_kernel<<<nq, 128, 0, s>>>(keys, counts, k, thr, cand, cap, ccount);
    count_launch();
}
}  // namespace pb
