// kernels_rescue.cu -- exact fallback for candidate-list overflow (K2x flat, K6x IVF).
//
// The scans append every key below a query's running bound thr[q] to that query's
// candidate list (capacity cap).  Ordinary inputs stay far below cap because thr
// tightens as the scan proceeds, but a database ordered adversarially (keys
// arriving in descending order, e.g. sorted by falling ADC to the query) defeats
// the tightening and fills the list.  Such a query is flagged (ovq[q]) instead of
// dropping keys silently; before its final top-k (K3) the rescue scan re-ranks
// it exactly with bounded memory: each CTA streams its slice of the query's
// codes, keeps every key below a local bound in a shared-memory buffer and, when
// the buffer fills, radix-selects the buffer's k-th key, lowers the local bound
// to it and compacts -- the top-k contract holds for any
// arrival order.  The CTA's final top-k replaces the query's candidate list
// (parts of <= k keys appended at rcount[q]), and K3 ranks the union exactly.
// Queries that did not overflow cost one flag load per CTA.
#include <algorithm>

#include "code_ops.cuh"

namespace pb {

constexpr uint32_t RS_THREADS = 256;
constexpr uint32_t RS_BUF = 8192;  // keys per buffer (>= 2 x KMAX + one step of appends)

// k-th smallest (1-based, kk <= n) of n keys in shared memory: 8 passes of 8-bit
// digits, block-wide (RS_THREADS threads).
__device__ unsigned long long block_select_kth(const unsigned long long* keys, uint32_t n, uint32_t kk,
                                               uint32_t* hist, unsigned long long* prefix_s, uint32_t* want_s) {
    unsigned long long prefix = 0, mask = 0;
    uint32_t want = kk;
    for (int shift = 56; shift >= 0; shift -= 8) {
        hist[threadIdx.x] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += RS_THREADS) {
            const unsigned long long v = keys[i];
            if ((v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 0xFFu], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const uint32_t lane = threadIdx.x;
            uint32_t c[8], t = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) { c[j] = hist[lane * 8 + j]; t += c[j]; }
            uint32_t incl = t;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= (uint32_t)off) incl += o;
            }
            const uint32_t excl = incl - t;
            if (excl < want && want <= incl) {
                uint32_t r = want - excl;
                int digit = lane * 8 + 7;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (r <= c[j]) { digit = lane * 8 + j; break; }
                    r -= c[j];
                }
                *prefix_s = prefix | ((unsigned long long)digit << shift);
                *want_s = r;
            }
        }
        __syncthreads();
        prefix = *prefix_s;
        want = *want_s;
        mask |= 0xFFull << shift;
    }
    return prefix;
}

// Streaming top-k state of one CTA: keys below `bound` in buf[0, cnt).
struct RsState {
    unsigned long long* buf;  // RS_BUF keys
    unsigned long long* tmp;  // RS_BUF keys (compaction target)
    uint32_t* cnt;
    uint32_t* hist;
    unsigned long long* prefix;
    uint32_t* want;
    unsigned long long* bound;
};

// Keep the keys <= the k-th smallest (k distinct keys; duplicated ids may keep a few
// more).  Block-wide; leaves the result in buf and tightens the bound.
__device__ void rs_shrink(RsState& st, uint32_t k) {
    const uint32_t n = *st.cnt;
    if (n <= k) return;
    const unsigned long long kth = block_select_kth(st.buf, n, k, st.hist, st.prefix, st.want);
    __syncthreads();
    if (threadIdx.x == 0) *st.cnt = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += RS_THREADS) {
        const unsigned long long v = st.buf[i];
        if (v <= kth) st.tmp[atomicAdd(st.cnt, 1u)] = v;
    }
    __syncthreads();
    const uint32_t m = min(*st.cnt, RS_BUF / 2);
    for (uint32_t i = threadIdx.x; i < m; i += RS_THREADS) st.buf[i] = st.tmp[i];
    if (threadIdx.x == 0) {
        *st.cnt = m;
        if (kth + 1 < *st.bound) *st.bound = kth + 1;  // keys >= kth + 1 can no longer enter
    }
    __syncthreads();
}

// One step of appends (at most one key per thread), then shrink if the buffer nears full.
__device__ __forceinline__ void rs_offer(RsState& st, bool has, unsigned long long key, uint32_t k) {
    if (has && key < *st.bound) st.buf[atomicAdd(st.cnt, 1u)] = key;
    __syncthreads();
    if (*st.cnt > RS_BUF - RS_THREADS) rs_shrink(st, k);
}

// Flat (K2x): CTA s of S scans codes [n s / S, n (s + 1) / S) of every flagged query.
template <int M, int STRAT>
__global__ void __launch_bounds__(RS_THREADS) rescue_scan_kernel(const ScanArgs a, uint32_t* __restrict__ rcount) {
    using C = typename CodeT<M>::T;
    extern __shared__ __align__(16) uint8_t rs_smem[];
    float* lut = reinterpret_cast<float*>(rs_smem);
    __shared__ uint32_t cnt, hist[256], want;
    __shared__ unsigned long long prefix, bound;
    RsState st{reinterpret_cast<unsigned long long*>(rs_smem + M * KSUB * 4),
               reinterpret_cast<unsigned long long*>(rs_smem + M * KSUB * 4) + RS_BUF, &cnt, hist, &prefix, &want,
               &bound};
    constexpr bool USE_LUT = (STRAT == DUAL || STRAT == ADC);
    const uint64_t lo = a.n * blockIdx.x / gridDim.x, hi = a.n * (blockIdx.x + 1) / gridDim.x;
    {  // the common case -- no query overflowed -- costs one parallel pass over the flags
        uint32_t any = 0;
        for (uint32_t q = threadIdx.x; q < a.nqb; q += RS_THREADS) any |= __ldcg(a.ovq + q);
        if (!__syncthreads_or((int)any)) return;
    }
    for (uint32_t q = 0; q < a.nqb; ++q) {
        if (!__ldcg(a.ovq + q)) continue;  // uniform across the CTA
        __syncthreads();
        if (USE_LUT)
            for (uint32_t i = threadIdx.x; i < (uint32_t)M * KSUB; i += RS_THREADS)
                lut[i] = __ldg(a.lutp + (size_t)q * M * KSUB + i);
        const C qc = reinterpret_cast<const C*>(a.qcodes)[q];
        if (threadIdx.x == 0) {
            cnt = 0;
            bound = __ldcg(a.thr + q);  // a valid upper bound of the final k-th key
        }
        __syncthreads();
        for (uint64_t base = lo; base < hi; base += RS_THREADS) {
            const uint64_t pos = base + threadIdx.x;
            bool has = false;
            unsigned long long key = 0;
            if (pos < hi) {
                const C code = __ldg(reinterpret_cast<const C*>(a.codes) + pos);
                float score;
                if (strategy_score<M, STRAT>(lut, code, qc, a.tau, (uint32_t)(bound >> 32), score)) {
                    key = ((unsigned long long)__float_as_uint(score) << 32) |
                          (a.id_mode == ID_ARITH ? a.id0 + (uint32_t)pos : __ldg(a.id32 + pos));
                    has = true;
                }
            }
            rs_offer(st, has, key, a.k);
        }
        rs_shrink(st, a.k);
        __shared__ uint32_t at;
        if (threadIdx.x == 0) at = atomicAdd(rcount + q, cnt);
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < cnt; i += RS_THREADS)
            if (at + i < a.cap) a.cand[(size_t)q * a.cap + at + i] = st.buf[i];
    }
}

// ccount[q] = rcount[q] for the rescued queries (their lists were rewritten).
__global__ void rescue_fix_kernel(const uint32_t* __restrict__ ovq, const uint32_t* __restrict__ rcount, uint32_t nq,
                                  uint32_t cap, uint32_t* __restrict__ ccount) {
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x)
        if (ovq[q]) ccount[q] = min(rcount[q], cap);
}

template <int M, int STRAT>
static void launch_rescue_m(const ScanArgs& a, uint32_t* rcount, int num_sms, cudaStream_t s) {
    const size_t smem = (size_t)M * KSUB * 4 + 2 * (size_t)RS_BUF * 8;
    auto kfn = rescue_scan_kernel<M, STRAT>;
    set_max_smem((const void*)kfn, smem);
    // S CTAs, each contributing <= k keys: S * k <= cap (cap >= 128 k, capi.cu)
    const uint32_t S = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>({(uint64_t)num_sms, 128, a.cap / std::max(a.k, 1u)}));
    kfn<<<S, RS_THREADS, smem, s>>>(a, rcount);
    count_launch();
    rescue_fix_kernel<<<1, 256, 0, s>>>(a.ovq, rcount, a.nqb, a.cap, a.ccount);
    count_launch();
}

void launch_rescue(const ScanArgs& a, int strategy, uint32_t m, uint32_t* rcount, int num_sms, cudaStream_t s) {
    if (a.nqb == 0 || a.k == 0) return;
    const bool w = m == 16;
    switch (strategy) {
        case DUAL: w ? launch_rescue_m<16, DUAL>(a, rcount, num_sms, s) : launch_rescue_m<8, DUAL>(a, rcount, num_sms, s); break;
        case ADC: w ? launch_rescue_m<16, ADC>(a, rcount, num_sms, s) : launch_rescue_m<8, ADC>(a, rcount, num_sms, s); break;
        case BINARY:
            w ? launch_rescue_m<16, BINARY>(a, rcount, num_sms, s) : launch_rescue_m<8, BINARY>(a, rcount, num_sms, s);
            break;
        default:
            w ? launch_rescue_m<16, DISIDX>(a, rcount, num_sms, s) : launch_rescue_m<8, DISIDX>(a, rcount, num_sms, s);
            break;
    }
}

// IVF (K6x): persistent CTAs; each takes the flagged queries q = blockIdx.x (mod gridDim.x)
// and re-scans every visited probe (np_eff[q]) with that probe's residual LUT and query
// code, rewriting the query's candidate list.
template <int M, int STRAT>
__global__ void __launch_bounds__(RS_THREADS) ivf_rescue_kernel(const IvfScanArgs a, const uint32_t* __restrict__ np_eff,
                                                                uint32_t k) {
    using C = typename CodeT<M>::T;
    extern __shared__ __align__(16) uint8_t rs_smem[];
    float* lut = reinterpret_cast<float*>(rs_smem);
    __shared__ uint32_t cnt, hist[256], want;
    __shared__ unsigned long long prefix, bound;
    RsState st{reinterpret_cast<unsigned long long*>(rs_smem + M * KSUB * 4),
               reinterpret_cast<unsigned long long*>(rs_smem + M * KSUB * 4) + RS_BUF, &cnt, hist, &prefix, &want,
               &bound};
    constexpr bool USE_LUT = (STRAT == DUAL || STRAT == ADC);
    {  // the common case -- none of this CTA's queries overflowed -- costs one parallel pass over their flags
        uint32_t any = 0;
        for (uint64_t q = blockIdx.x + (uint64_t)threadIdx.x * gridDim.x; q < a.nq; q += (uint64_t)RS_THREADS * gridDim.x)
            any |= __ldcg(a.ovq + q);
        if (!__syncthreads_or((int)any)) return;
    }
    for (uint32_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
    if (!__ldcg(a.ovq + q)) continue;  // uniform across the CTA
    __syncthreads();
    if (threadIdx.x == 0) {
        cnt = 0;
        bound = a.thr[q];
    }
    const uint32_t ne = np_eff[q];
    for (uint32_t p = 0; p < ne; ++p) {
        const size_t item = (size_t)q * a.nprobe + p;
        const uint32_t cell = (uint32_t)a.probe_keys[item];
        __syncthreads();
        if (USE_LUT)
            for (uint32_t i = threadIdx.x; i < (uint32_t)M * KSUB; i += RS_THREADS) lut[i] = a.lutp[item * M * KSUB + i];
        const C qc = reinterpret_cast<const C*>(a.qcodes)[item];
        __syncthreads();
        const uint64_t lo = a.off[cell], hi = a.off[cell + 1];
        for (uint64_t base = lo; base < hi; base += RS_THREADS) {
            const uint64_t pos = base + threadIdx.x;
            bool has = false;
            unsigned long long key = 0;
            if (pos < hi) {
                const C code = reinterpret_cast<const C*>(a.codes)[pos];
                float score;
                if (strategy_score<M, STRAT>(lut, code, qc, a.tau, (uint32_t)(bound >> 32), score)) {
                    key = ((unsigned long long)__float_as_uint(score) << 32) | a.low[pos];
                    has = true;
                }
            }
            rs_offer(st, has, key, k);
        }
    }
    rs_shrink(st, k);
    const uint32_t n = min(cnt, a.cap);
    for (uint32_t i = threadIdx.x; i < n; i += RS_THREADS) a.cand[(size_t)q * a.cap + i] = st.buf[i];
    if (threadIdx.x == 0) a.ccount[q] = n;
    }
}

template <int M, int STRAT>
static void launch_ivf_rescue_m(const IvfScanArgs& a, const uint32_t* np_eff, uint32_t k, cudaStream_t s) {
    const size_t smem = (size_t)M * KSUB * 4 + 2 * (size_t)RS_BUF * 8;
    auto kfn = ivf_rescue_kernel<M, STRAT>;
    set_max_smem((const void*)kfn, smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    kfn<<<std::min<uint32_t>(a.nq, (uint32_t)sms), RS_THREADS, smem, s>>>(a, np_eff, k);
    count_launch();
}

void launch_ivf_rescue(const IvfScanArgs& a, int strategy, uint32_t m, const uint32_t* np_eff, uint32_t k,
                       cudaStream_t s) {
    if (a.nq == 0 || k == 0) return;
    const bool w = m == 16;
    switch (strategy) {
        case DUAL: w ? launch_ivf_rescue_m<16, DUAL>(a, np_eff, k, s) : launch_ivf_rescue_m<8, DUAL>(a, np_eff, k, s); break;
        case ADC: w ? launch_ivf_rescue_m<16, ADC>(a, np_eff, k, s) : launch_ivf_rescue_m<8, ADC>(a, np_eff, k, s); break;
        case BINARY:
            w ? launch_ivf_rescue_m<16, BINARY>(a, np_eff, k, s) : launch_ivf_rescue_m<8, BINARY>(a, np_eff, k, s);
            break;
        default:
            w ? launch_ivf_rescue_m<16, DISIDX>(a, np_eff, k, s) : launch_ivf_rescue_m<8, DISIDX>(a, np_eff, k, s);
            break;
    }
}

}  // namespace pb
