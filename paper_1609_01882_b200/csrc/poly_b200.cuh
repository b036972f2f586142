// poly_b200.cuh -- shared device helpers and kernel entry points (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pb {

constexpr int KSUB = 256;              // dbits = 8
constexpr int DSUB = 16;               // every configuration: 128/8 and 256/16
#define POLY_STR2(x) #x
#define POLY_STR(x) POLY_STR2(x)
#ifndef POLY_WAIT_HINT  // mbarrier try_wait suspend-time hint (ns); 0 = none
#define POLY_WAIT_HINT 20000
#endif
#ifndef POLY_AFFINE  // 1: group-affine K2 schedule
#define POLY_AFFINE 1
#endif
#ifndef POLY_AFFINE_LEAD  // K2: chunks a query group may run ahead of the slowest one
#define POLY_AFFINE_LEAD 16
#endif
#ifndef POLY_UNITS_PER_CTA  // K2 work units per CTA the unit size aims for (capped by POLY_MAX_TPC)
#define POLY_UNITS_PER_CTA 16
#endif
#ifndef POLY_MAX_TPC  // tiles per K2 work unit (cap): fewer unit boundaries vs. tail balance
#define POLY_MAX_TPC 128
#endif
#ifndef POLY_SEL_BS  // candidate-list slots per threshold select (>= 4k)
#define POLY_SEL_BS 512
#endif
#ifndef POLY_SEL_KF  // select block >= KF * k slots
#define POLY_SEL_KF 4
#endif
#ifndef POLY_SEED_BLOCKS  // K2s seed sample: runs of 256 codes (0 = no seed kernel)
#define POLY_SEED_BLOCKS 128
#endif
#ifndef POLY_SPIN_MMA_NS  // K2: backoff of the quad-MMA commit wait
#define POLY_SPIN_MMA_NS 400
#endif
#ifndef POLY_SPIN_NS
#define POLY_SPIN_NS 400
#endif
#ifndef POLY_TILE_BYTES
#define POLY_TILE_BYTES 14336
#endif
#ifndef POLY_STAGES
#define POLY_STAGES 4
#endif
constexpr int TILE_BYTES = POLY_TILE_BYTES;  // code bytes per pipeline stage (1536 codes at m = 8)
constexpr int STAGES = POLY_STAGES;          // bulk-copy ring depth
#ifndef POLY_SCAN_WARPS
#define POLY_SCAN_WARPS 28
#endif
constexpr int SCAN_WARPS = POLY_SCAN_WARPS;  // K2 consumer warps (plus one TMA producer warp)
constexpr int BS = 4096;               // candidate list capacity unit: a list holds >= 32 * BS keys per query
constexpr int KMAX = 2048;             // largest supported k
constexpr int MAXREQ = 32;             // pending threshold selects per CTA (ring)
constexpr uint64_t KEY_INF = ~0ull;

enum Strategy { ADC = 0, BINARY = 1, DISIDX = 2, DUAL = 3 };
enum IdMode { ID_ARITH = 0, ID_TABLE = 1 };  // key low word = id0 + pos, or id32[pos]

// Host/device argument block of the fused scan (K2).
struct ScanArgs {
    const uint8_t* codes;        // n x CB bytes, padded to a multiple of TILE codes
    uint64_t n;                  // codes in this shard
    const float* lutp;           // nqb x M x 256 (stored-field indexed LUTs)
    const uint8_t* qcodes;       // nqb x CB
    uint32_t nqb, tau, k;
    int id_mode;
    uint32_t id0;
    const uint32_t* id32;        // pos -> key low word (ID_TABLE)
    unsigned long long* cand;    // nqb x cap candidate keys
    uint32_t cap;
    uint32_t* ccount;            // nqb
    uint32_t* bdone;             // nqb x (cap / BS) completion counters
    unsigned long long* thr;     // nqb running upper bounds of the k-th key
    unsigned long long* surv;    // per-query survivor counts (per_query_stats) or [0] = batch total
    unsigned long long* surv_hash;  // per_query_stats: per-query sum of mix64(key low word) over survivors
    uint32_t* ovq;               // per query: set when a candidate did not fit (the rescue scan re-ranks it)
    uint32_t* work;              // dynamic work-unit counter
    uint32_t units, ngroups, tiles_per_chunk;
    // group-affine schedule (affine = 1): work[g] counts the chunks handed out of
    // query group g; a CTA stays on its group (no LUT reload) until it runs dry
    uint32_t affine, nchunks;
    uint64_t ntiles;             // logical tiles; physical tile = logical * tile_stride
    uint64_t tile_stride;
    uint32_t bs;                 // candidate block size (>= k) for threshold selects
};

// Argument block of the IVF list scan (K6).
struct IvfScanArgs {
    const uint8_t* codes;                 // list-ordered residual codes
    const uint32_t* low;                  // list-ordered key low words (id or id rank)
    const uint64_t* off;                  // nlist + 1 list offsets
    const unsigned long long* probe_keys; // nq x nprobe (dist bits << 32 | cell), ascending
    const float* lutp;                    // (nq x nprobe) x M x 256 residual LUTs
    const uint8_t* qcodes;                // (nq x nprobe) x CB residual query codes
    uint32_t nq, nprobe, tau;
    unsigned long long* thr;              // per-query key bound (seeded between rounds)
    unsigned long long* cand;             // nq x cap candidate keys
    uint32_t cap;
    uint32_t* ccount;
    uint32_t* ovq;                        // per query: a candidate did not fit (rescued before the final K3)
    uint32_t* work;
    unsigned long long* surv_total;
    unsigned long long* surv_q;           // per-query survivor counts and hashes (stats mode; else null)
    unsigned long long* hash_q;
    const uint4* items;      // work items (query, probe, pos, rows): `rows` codes from list-order position
    const uint32_t* nitems;  // `pos` (a chunk of the probed cell's list); built by the probe-count kernel
    uint32_t items_cap;
};

// Work lists of the two K6 rounds, written by launch_ivf_probe_count.
struct IvfWork {
    uint4* items[2];
    uint32_t* nitems;   // 2 counters (zeroed before the launch)
    uint32_t cap[2];
    uint32_t chunk[2];
    uint32_t* overflow;
    // the (query, probe) items of each round whose list is not empty here: the residual
    // LUTs K1r builds (by-list sharding leaves most lists of a rank empty)
    uint32_t* lut_items[2];
    uint32_t* nlut;     // 2 counters (zeroed)
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
#if POLY_WAIT_HINT > 0
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, " POLY_STR(POLY_WAIT_HINT) ";\n"
#else
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
#endif
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok;
}

// ---- tcgen05 / TMEM helpers (K2's tensor-core Hamming filter) ----
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {  // one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // one full warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// 32 lanes x 16 columns (one register per column) of the warp's lane quadrant
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, uint32_t v) {  // 8 columns of one value
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// D[tmem] (+)= A[tmem] . B[smem desc], kind::i8 (s8 x s8 -> s32)
__device__ __forceinline__ void mma_i8_ts(uint32_t d_t, uint32_t a_t, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_t),
        "r"(a_t), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Wait with a timer backoff (POLY_SPIN_NS > 0): a suspended try_wait wakes on any
// mbarrier activity in the CTA, which a 25-warp K2 has plenty of.
template <uint32_t NS = POLY_SPIN_NS>
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
    if constexpr (NS > 0) {
        while (!mbar_test(bar, parity)) __nanosleep(NS);
    } else {
        mbar_wait(bar, parity);
    }
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// splitmix64 finaliser: survivor-set hash sum_i mix64(id_i) (order-independent;
// the oracle computes the same, oracle/polyoracle.c po_mix64)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------- kernels
// K1: LUT build + query code (compute_lut pq.cpp:91-105, permuted_lut :107-119, encode :29-45).
void launch_lut(const float* queries, uint32_t nq, uint32_t dim, uint32_t m, const float* codebooks,
                const uint16_t* perms, float* lutp, uint8_t* qcodes, cudaStream_t s);

// K0: DB encoder (encode pq.cpp:29-45 per vector), from device floats or the synthetic generator.
void launch_encode(const float* x, uint64_t n, uint32_t dim, uint32_t m, const float* codebooks,
                   const uint16_t* perms, uint8_t* codes, cudaStream_t s);
void launch_synth_encode(uint64_t seed, uint32_t stream_id, uint64_t row0, uint64_t n, const float* centers,
                         uint32_t ncent, uint32_t dim, int normalize, uint32_t m, const float* codebooks,
                         const uint16_t* perms, uint8_t* codes, cudaStream_t s);
void launch_gen_points(uint64_t seed, uint32_t stream_id, uint64_t row0, uint64_t n, const float* centers,
                       uint32_t ncent, uint32_t dim, int normalize, float* out, cudaStream_t s);

// K2: fused filter + ADC + candidate scan.
void launch_scan(const ScanArgs& a, int strategy, uint32_t m, bool per_query_stats, int num_sms, cudaStream_t s);
int scan_queries_per_cta(uint32_t m);
// K2s: thr[q] = min(thr[q], k-th key of a fixed sample + 1); one CTA per query
void launch_seed_sample(const ScanArgs& a, int strategy, uint32_t m, uint32_t nq, uint32_t seed_blocks, cudaStream_t s);

// K3: per-query exact top-k over candidate keys; K3b: key -> (id, score).
// cand part p, query q: cand + p * part_stride + q * cap, count ccount[p * count_stride + q].
void launch_topk(const unsigned long long* cand, const uint32_t* ccount, uint32_t cap, uint32_t parts,
                 uint64_t part_stride, uint64_t count_stride, uint32_t nq, uint32_t k, unsigned long long* out_keys,
                 uint32_t* out_counts, cudaStream_t s);
void launch_keys_to_ids(const unsigned long long* keys, const uint32_t* counts, uint32_t nq, uint32_t k,
                        const int64_t* rank_to_id, int64_t* out_ids, float* out_scores, uint32_t* out_counts,
                        cudaStream_t s);

// Calibration: Hamming histograms (nq x (code_bits + 1)).
void launch_hamming_hist(const uint8_t* codes, uint64_t n, uint32_t cb, const uint8_t* qcodes, uint32_t nq,
                         unsigned long long* hist, cudaStream_t s);
// with_assignments: relabel fields through a per-sub-quantizer byte map.
void launch_relabel(uint8_t* codes, uint64_t n, uint32_t m, const uint8_t* maps, cudaStream_t s);

void launch_seed_compact(const unsigned long long* keys, const uint32_t* counts, uint32_t nq, uint32_t k,
                         unsigned long long* thr, unsigned long long* cand, uint32_t cap, uint32_t* ccount,
                         cudaStream_t s);
// IVF (kernels_ivf.cu)
void launch_coarse_keys(const float* q, uint32_t nq, uint32_t dim, const float* cent, uint32_t nlist,
                        unsigned long long* keys, cudaStream_t s);
// K5t + K5q (kernels_coarse.cu): enumerate_cells on the tensor cores, exact, np <= coarse_rank_npmax()
uint32_t coarse_tc_tiles(uint32_t nlist);
uint32_t coarse_rank_npmax();
void launch_coarse_pack(const float* cent, uint32_t nlist, uint32_t dim, float* packed, float* cnorm_pad,
                        cudaStream_t s);
void launch_coarse_tc(const float* q, uint32_t nq, uint32_t dim, const float* packed, const float* cnorm_pad,
                      uint32_t nlist, int num_sms, float4* grp, cudaStream_t s);
void launch_coarse_rank(const float* q, uint32_t nq, uint32_t dim, const float4* grp, uint32_t nlist, float cmax,
                        const float* cent, uint32_t np, uint32_t* scratch, unsigned long long* probe_keys,
                        uint32_t* probe_counts, cudaStream_t s);
// K1r over a list of items (q * nprobe + p; count on the device, at most max_items)
void launch_residual_lut(const float* queries, uint32_t dim, uint32_t m, const unsigned long long* probe_keys,
                         uint32_t nprobe, const uint32_t* items, const uint32_t* nitems, uint32_t max_items,
                         const float* cent, const float* codebooks, const uint16_t* perms, float* lutp,
                         uint8_t* qcodes, cudaStream_t s);
void launch_ivf_probe_count(const unsigned long long* probe_keys, uint32_t nq, uint32_t nprobe, const uint64_t* off,
                            uint64_t cap, uint32_t* np_eff, unsigned long long* scanned, cudaStream_t s,
                            uint32_t* split, uint64_t r1_codes, uint32_t r1_max, const IvfWork& w);
void launch_ivf_scan(const IvfScanArgs& a, int strategy, uint32_t m, int num_sms, cudaStream_t s);
// K6s: round-1 bound from the first `rows` codes of each query's first probed list
void launch_ivf_seed(const IvfScanArgs& a, int strategy, uint32_t m, uint32_t rows, uint32_t k, cudaStream_t s);
void launch_assign(const float* x, uint64_t n, uint32_t dim, const float* cent, uint32_t nlist, uint32_t* assign,
                   cudaStream_t s);
void launch_residual_encode(const float* x, uint64_t n, uint32_t dim, uint32_t m, const float* cent,
                            const uint32_t* assign, const float* codebooks, const uint16_t* perms, uint8_t* codes,
                            cudaStream_t s);
void launch_cell_hist(const uint32_t* assign, uint64_t n, unsigned long long* hist, cudaStream_t s);
void launch_cell_scatter(const uint32_t* assign, uint64_t n, uint32_t cb, const uint8_t* codes_in,
                         const uint32_t* low_in, unsigned long long* cursor, uint8_t* codes_out, uint32_t* low_out,
                         cudaStream_t s);
void launch_key_low(uint64_t n, int mode, uint32_t id0, const uint32_t* id32, uint32_t* out, cudaStream_t s);
void launch_or_flag(uint32_t* dst, const uint32_t* src, cudaStream_t s);
void count_launch();
// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the current device (the
// attribute is per device context: tracked per (kernel, device), thread-safe)
void set_max_smem(const void* fn, size_t bytes);
// K2x / K6x: exact re-rank of the queries whose candidate list overflowed (ovq[q]):
// streaming top-k over the query's codes, written back as its candidate list
void launch_rescue(const ScanArgs& a, int strategy, uint32_t m, uint32_t* rcount, int num_sms, cudaStream_t s);
void launch_ivf_rescue(const IvfScanArgs& a, int strategy, uint32_t m, const uint32_t* np_eff, uint32_t k,
                       cudaStream_t s);

}  // namespace pb
