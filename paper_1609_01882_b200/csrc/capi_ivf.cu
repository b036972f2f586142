// capi_ivf.cu -- C ABI of the IVF search path (include/poly_b200.h, poly_b200_ivf_*).
//
// Restates the SPEC's coarseindex module (the reference has
// no code for it) on the GPU: build = exact nearest-cell assignment + residual
// encode + CSR lists; search_coarse = K5 (coarse keys) -> K3 (nprobe nearest
// cells) -> K1r (per-(query, cell) residual LUTs and codes) -> rounds of K6
// list scans over probes [0,1), [1,4), [4,16), ... with the k-th key of the
// candidates so far (K3) seeding each next round's threshold -> K3 top-k.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "../../include/poly_b200.h"
#include "host_common.h"
#include "poly_b200.cuh"

using namespace pbh;

#ifndef POLY_IVF_NQB
#define POLY_IVF_NQB 2048
#endif
namespace {
constexpr uint32_t IVF_NQB = POLY_IVF_NQB;  // queries per batch
}

struct poly_b200_ivf {
    int device = 0;
    int num_sms = 148;
    uint32_t m = 0, dim = 0, cb = 0, nlist = 0;
    std::vector<float> h_codebooks, h_coarse;
    std::vector<uint16_t> h_perms;
    float* d_codebooks = nullptr;
    uint16_t* d_perms = nullptr;
    float* d_coarse = nullptr;

    // insertion-order staging
    uint8_t* d_codes_ins = nullptr;
    uint32_t* d_cells_ins = nullptr;
    uint64_t n = 0, cap_ins = 0;
    pbh::IdMap idm;

    // CSR lists (rebuilt lazily after adds)
    bool lists_dirty = true;
    std::vector<uint64_t> h_off;
    uint64_t* d_off = nullptr;
    uint8_t* d_codes_list = nullptr;
    uint32_t* d_low_list = nullptr;
    uint64_t max_list = 0;

    // search scratch
    uint32_t nqb = IVF_NQB;               // queries per batch (poly_b200_ivf_set_batch)
    unsigned long long* ckeys = nullptr;  // K5 (nprobe > 1024): nqb x nlist exact keys (lazy)
    uint32_t* nl_counts = nullptr;         // K3 counts of K5: nlist per query
    float4* grp = nullptr;                 // K5t: per (group of 128 cells, query) kept values
    uint32_t* rank_scratch = nullptr;      // K5q: per-query candidate cells (nqb x nlist)
    unsigned long long* probe_keys = nullptr;
    uint32_t* probe_counts = nullptr;
    uint32_t* np_eff = nullptr;
    uint32_t* split = nullptr;  // per query: probes of round 1
    unsigned long long* scanned = nullptr;
    uint32_t scratch_nprobe = 0;
    uint4* items[2] = {nullptr, nullptr};  // K6 work lists of the two rounds
    uint32_t* lut_items = nullptr;         // K1r item lists of the two rounds (2 x nqb x np)
    uint64_t items_cap[2] = {0, 0};
    float* lutp = nullptr;
    uint8_t* qcodes = nullptr;
    unsigned long long* cand = nullptr;
    uint32_t cand_cap = 0;
    uint32_t cap_override = 0;  // test hook: candidate-list capacity (0 = the default)
    uint32_t* ctrl = nullptr;  // [ccount NQB][overflow][work x 16]
    unsigned long long* thr = nullptr;
    unsigned long long* keys = nullptr;
    uint32_t keys_k = 0;
    uint32_t* kcounts = nullptr;
    unsigned long long* surv_total = nullptr;
    unsigned long long* scan_total = nullptr;
    uint32_t* ovq = nullptr;                 // per query: candidate list overflowed (rescued)
    unsigned long long* surv_q = nullptr;    // per-query survivor counts / hashes (stats mode)
    unsigned long long* hash_q = nullptr;
    uint32_t* sticky_overflow = nullptr;     // work-list overflow (an internal invariant)
    uint32_t* h_overflow = nullptr;          // pinned copy, checked at the next call
    cudaEvent_t done_ev = nullptr;
    bool pending_check = false;
    bool phase_pending = false, phase_empty = false;  // two-phase search state (phase 1 done)
    uint64_t phase_nq = 0;
    float* d_q = nullptr;
    uint64_t d_q_cap = 0;
    int64_t* d_oid = nullptr;
    float* d_osc = nullptr;
    uint32_t* d_ocnt = nullptr;
    uint64_t d_out_rows = 0;
    uint32_t d_out_k = 0;

    // knn_graph staging (k + 1 results per row)
    int64_t* knn_ids = nullptr;
    float* knn_sc = nullptr;
    uint32_t* knn_cnt = nullptr;
    uint64_t knn_rows = 0;
    uint32_t knn_k1 = 0;

    // K5t/K5q (tensor-core coarse quantization): the centroids packed into 32 KB stage
    // images, |c|^2 per cell (+inf past nlist), an upper bound of |c|
    float* d_cpacked = nullptr;
    float* d_cnorm = nullptr;
    float cmax = 0.0f;

    // K6 timing (bench.py): CUDA events around every list-scan launch on its stream
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    size_t prof_used = 0;

    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // K1r of the round-2 probes, overlapping round 1
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::mutex mu;
    uint32_t code_bits() const { return m * 8; }
};

namespace {

#ifndef POLY_IVF_R1_MAX
#define POLY_IVF_R1_MAX 2
#endif
#ifndef POLY_IVF_R1_CODES
#define POLY_IVF_R1_CODES 2048
#endif
constexpr uint32_t IVF_R1_MAX = POLY_IVF_R1_MAX;      // round 1: at most this many leading probes
constexpr uint64_t IVF_R1_CODES = POLY_IVF_R1_CODES;  // ... and at least this many codes
#ifndef POLY_IVF_CHUNK2
#define POLY_IVF_CHUNK2 4096
#endif
#ifndef POLY_IVF_CHUNK
#define POLY_IVF_CHUNK 4096
#endif
constexpr uint32_t IVF_CHUNK = POLY_IVF_CHUNK;    // K6 round-1 work item: rows of a list (A/B with the unit pipeline: 512 / 1024 / 2048 / 4096 / 8192 rows -> 924 / 760 / 676 / 665 / 695 us)
constexpr uint32_t IVF_CHUNK2 = POLY_IVF_CHUNK2;  // round 2: longer items (fewer LUT loads per code)
#ifndef POLY_IVF_SEED_ROWS  // K6s sample: rows of each query's first list (0 = no round-1 seed)
#define POLY_IVF_SEED_ROWS 2048
#endif
constexpr uint32_t IVF_SEED_ROWS = POLY_IVF_SEED_ROWS;

__global__ void fill_u32(uint32_t* p, uint64_t n, uint32_t v) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void add_u64(const unsigned long long* src, uint32_t n, unsigned long long* dst) {
    unsigned long long s = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) s += src[i];
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(dst, s);
}

__global__ void probes_to_cells(const unsigned long long* keys, uint64_t n, uint32_t* cells) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        cells[i] = (uint32_t)keys[i];
}

void grow_ins(poly_b200_ivf* iv, uint64_t need) {
    if (need <= iv->cap_ins) return;
    const uint64_t cap = std::max<uint64_t>(need, iv->cap_ins * 2);
    uint8_t* c = dalloc<uint8_t>(cap * iv->cb);
    uint32_t* a = dalloc<uint32_t>(cap);
    if (iv->n) {
        CK(cudaMemcpyAsync(c, iv->d_codes_ins, iv->n * iv->cb, cudaMemcpyDeviceToDevice, iv->stream));
        CK(cudaMemcpyAsync(a, iv->d_cells_ins, iv->n * 4, cudaMemcpyDeviceToDevice, iv->stream));
    }
    CK(cudaStreamSynchronize(iv->stream));
    dfree(iv->d_codes_ins);
    dfree(iv->d_cells_ins);
    iv->d_codes_ins = c;
    iv->d_cells_ins = a;
    iv->cap_ins = cap;
}

// CSR rebuild: histogram of cells -> offsets -> scatter codes and key-low words.
void rebuild_lists(poly_b200_ivf* iv) {
    if (!iv->lists_dirty) return;
    cudaStream_t s = iv->stream;
    // list positions are 32-bit in the K6 work items and the key low words
    require(iv->n < (1ull << 32), POLY_B200_INVALID_ARGUMENT, "an IVF index holds < 2^32 codes per GPU");
    iv->idm.sync(iv->n);
    dfree(iv->d_codes_list);
    dfree(iv->d_low_list);
    const uint64_t pad = 1024;
    iv->d_codes_list = dalloc<uint8_t>((iv->n + pad) * iv->cb);
    iv->d_low_list = dalloc<uint32_t>(iv->n + pad);
    unsigned long long* hist = dalloc<unsigned long long>(iv->nlist);
    uint32_t* low_ins = dalloc<uint32_t>(std::max<uint64_t>(iv->n, 1));
    try {
        CK(cudaMemsetAsync(hist, 0, iv->nlist * 8, s));
        pb::launch_cell_hist(iv->d_cells_ins, iv->n, hist, s);
        std::vector<unsigned long long> h(iv->nlist);
        CK(cudaMemcpyAsync(h.data(), hist, iv->nlist * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        iv->h_off.assign(iv->nlist + 1, 0);
        iv->max_list = 0;
        for (uint32_t c = 0; c < iv->nlist; ++c) {
            iv->h_off[c + 1] = iv->h_off[c] + h[c];
            iv->max_list = std::max<uint64_t>(iv->max_list, h[c]);
        }
        CK(cudaMemcpyAsync(iv->d_off, iv->h_off.data(), (iv->nlist + 1) * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(hist, iv->h_off.data(), iv->nlist * 8, cudaMemcpyHostToDevice, s));  // cursors
        pb::launch_key_low(iv->n, iv->idm.mode, iv->idm.key_id0, iv->idm.d_id32, low_ins, s);
        pb::launch_cell_scatter(iv->d_cells_ins, iv->n, iv->cb, iv->d_codes_ins, low_ins, hist, iv->d_codes_list,
                                iv->d_low_list, s);
        CK(cudaStreamSynchronize(s));
        CK(cudaGetLastError());
    } catch (...) {
        dfree(hist);
        dfree(low_ins);
        throw;
    }
    dfree(hist);
    dfree(low_ins);
    iv->lists_dirty = false;
}

void ensure_ivf_scratch(poly_b200_ivf* iv, uint32_t nprobe, uint32_t k) {
    if (!iv->np_eff) {
        iv->grp = dalloc<float4>((size_t)iv->nqb * 2 * pb::coarse_tc_tiles(iv->nlist));
        iv->rank_scratch = dalloc<uint32_t>((size_t)iv->nqb * iv->nlist);
        iv->np_eff = dalloc<uint32_t>(iv->nqb);
        iv->split = dalloc<uint32_t>(iv->nqb);
        iv->scanned = dalloc<unsigned long long>(iv->nqb);
        iv->ctrl = dalloc<uint32_t>(iv->nqb + 32);
        iv->thr = dalloc<unsigned long long>(iv->nqb);
        iv->kcounts = dalloc<uint32_t>(iv->nqb);
        iv->surv_total = dalloc<unsigned long long>(1);
        iv->scan_total = dalloc<unsigned long long>(1);
        iv->ovq = dalloc<uint32_t>(iv->nqb);
        iv->surv_q = dalloc<unsigned long long>(iv->nqb);
        iv->hash_q = dalloc<unsigned long long>(iv->nqb);
        iv->sticky_overflow = dalloc<uint32_t>(1);
        CK(cudaMallocHost(&iv->h_overflow, sizeof(uint32_t)));
        *iv->h_overflow = 0;
        CK(cudaEventCreateWithFlags(&iv->done_ev, cudaEventDisableTiming));
    }
    if (iv->scratch_nprobe < nprobe) {
        dfree(iv->probe_keys);
        dfree(iv->probe_counts);
        dfree(iv->lutp);
        dfree(iv->qcodes);
        iv->scratch_nprobe = nprobe;
        iv->probe_keys = dalloc<unsigned long long>((size_t)iv->nqb * nprobe);
        iv->probe_counts = dalloc<uint32_t>(iv->nqb);
        iv->lutp = dalloc<float>((size_t)iv->nqb * nprobe * iv->m * 256);
        iv->qcodes = dalloc<uint8_t>((size_t)iv->nqb * nprobe * iv->cb);
        dfree(iv->lut_items);
        iv->lut_items = dalloc<uint32_t>((size_t)2 * iv->nqb * nprobe);
    }
    const uint64_t r1 = std::min<uint64_t>(nprobe, IVF_R1_MAX);
    // work-list bounds per query: round 1 <= r1 probes -> <= r1 + r1 * max_list / CHUNK items;
    // round 2 <= np + min(n, np * max_list) / CHUNK2 items
    const uint64_t need[2] = {
        (uint64_t)iv->nqb * (r1 + (r1 * iv->max_list + IVF_CHUNK - 1) / IVF_CHUNK),
        (uint64_t)iv->nqb * (nprobe + r1 + (std::min<uint64_t>(iv->n, nprobe * iv->max_list) + IVF_CHUNK2 - 1) / IVF_CHUNK2)};
    for (int r = 0; r < 2; ++r)
        if (iv->items_cap[r] < need[r]) {
            require(need[r] < (1ull << 32), POLY_B200_INVALID_ARGUMENT, "IVF work list too large");
            dfree(iv->items[r]);
            iv->items_cap[r] = need[r];
            iv->items[r] = dalloc<uint4>(need[r]);
        }
    // Round 2 is bounded by round 1's k-th key.  Round 1 is bounded by the K6s seed when it runs
    // (k <= IVF_SEED_ROWS / 4): 131,072 keys then hold its candidates with a wide margin.  Without the
    // seed round 1 has no bound and its <= r1 probes' survivors must fit.  A list that still fills up
    // (a query whose seed found fewer than k keys and whose next list is huge) is re-ranked by the
    // exact rescue scan.
    const bool seeded = IVF_SEED_ROWS && k <= IVF_SEED_ROWS / 4;
    uint32_t cap = (uint32_t)std::max<uint64_t>(131072, seeded ? 4ull * k : r1 * iv->max_list + k);
    if (iv->cap_override) cap = std::max<uint32_t>(iv->cap_override, k);
    if (iv->cand_cap != cap) {
        dfree(iv->cand);
        iv->cand_cap = cap;
        iv->cand = dalloc<unsigned long long>((size_t)iv->nqb * cap);
    }
    if (iv->keys_k < k) {
        dfree(iv->keys);
        iv->keys_k = k;
        iv->keys = dalloc<unsigned long long>((size_t)iv->nqb * k);
    }
}

void validate(const poly_b200_ivf* iv, const poly_b200_ivf_params* p) {
    require(p != nullptr, POLY_B200_INVALID_ARGUMENT, "null search params");
    require(p->strategy >= 0 && p->strategy <= 3, POLY_B200_INVALID_ARGUMENT, "unknown strategy");
    require(p->tau <= iv->code_bits(), POLY_B200_INVALID_ARGUMENT, "tau exceeds code bits");
    require(p->k <= (uint32_t)pb::KMAX, POLY_B200_INVALID_ARGUMENT, "k > 2048 is not supported on the GPU path");
    require(p->nprobe >= 1, POLY_B200_INVALID_ARGUMENT, "nprobe must be >= 1");  // CoarseConfig: nprobe >= 1
    // enumerate_cells ranks min(nprobe, nlist) cells per query with K3 (k <= KMAX)
    require(std::min(p->nprobe, iv->nlist) <= (uint32_t)pb::KMAX, POLY_B200_INVALID_ARGUMENT,
            "min(nprobe, nlist) > 2048 is not supported on the GPU path");
}

// The work-list overflow flag of an earlier call (an internal invariant: the lists are
// sized to their bound); raised at the next call on this index.
void check_pending(poly_b200_ivf* iv, bool wait) {
    if (!iv->pending_check) return;
    if (wait) CK(cudaEventSynchronize(iv->done_ev));
    else if (cudaEventQuery(iv->done_ev) != cudaSuccess) return;
    iv->pending_check = false;
    if (*iv->h_overflow) {
        *iv->h_overflow = 0;
        throw Error(POLY_B200_INTERNAL, "IVF work list overflow in a previous search: its results are incomplete");
    }
}

// Enqueue enumerate_cells for a batch: probe_keys (nqb x np) ascending.
// np <= 1024: tensor-core dots with the per-group kept values (K5t) and the exact re-rank
// of the cells within the error bound (K5q); larger np: every exact key (K5), then K3.
void enumerate_cells(poly_b200_ivf* iv, const float* d_q, uint32_t nqb, uint32_t np, cudaStream_t s) {
    if (np <= pb::coarse_rank_npmax()) {
        pb::launch_coarse_tc(d_q, nqb, iv->dim, iv->d_cpacked, iv->d_cnorm, iv->nlist, iv->num_sms, iv->grp, s);
        pb::launch_coarse_rank(d_q, nqb, iv->dim, iv->grp, iv->nlist, iv->cmax, iv->d_coarse, np, iv->rank_scratch,
                               iv->probe_keys, iv->probe_counts, s);
        return;
    }
    if (!iv->ckeys) {
        iv->ckeys = dalloc<unsigned long long>((size_t)iv->nqb * iv->nlist);
        iv->nl_counts = dalloc<uint32_t>(iv->nqb);
        fill_u32<<<1, 256, 0, s>>>(iv->nl_counts, iv->nqb, iv->nlist);
        pb::count_launch();
    }
    pb::launch_coarse_keys(d_q, nqb, iv->dim, iv->d_coarse, iv->nlist, iv->ckeys, s);
    pb::launch_topk(iv->ckeys, iv->nl_counts, iv->nlist, 1, 0, 0, nqb, np, iv->probe_keys, iv->probe_counts, s);
}

// One batch of <= 256 queries; outputs through keys_to_ids.
__global__ void min_u64(unsigned long long* dst, const unsigned long long* src, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[i] = src[i] < dst[i] ? src[i] : dst[i];
}

// phase 0: the whole search.  Two-phase form (by-list sharding):
// phase 1 = round 1 over each query's FIRST probe only (empty here unless this rank owns
// it), its k-th key + 1 out as d_thr; the caller min-reduces the bounds over the ranks;
// phase 2 = round 2 (every other probe) under min(local, d_thr), then the final top-k.
void search_batch(poly_b200_ivf* iv, const float* d_q, uint32_t nqb, const poly_b200_ivf_params* p, int64_t* d_ids,
                  float* d_scores, uint32_t* d_counts, cudaStream_t s, uint64_t* d_keys_out = nullptr,
                  uint32_t* d_kcounts_out = nullptr, const uint64_t* d_probes_in = nullptr, uint64_t* d_surv = nullptr,
                  uint64_t* d_hash = nullptr, int phase = 0, uint64_t* d_thr = nullptr) {
    const uint32_t k = p->k;
    const uint32_t np = std::min(p->nprobe, iv->nlist);
    int strategy = p->strategy;
    if (strategy == pb::DUAL && p->tau >= iv->code_bits()) strategy = pb::ADC;  // SPEC.md:388 boundary
    const bool perq = d_surv || d_hash;
    if (phase != 2) {
        CK(cudaMemsetAsync(iv->ctrl, 0, (iv->nqb + 32) * 4, s));
        CK(cudaMemsetAsync(iv->ovq, 0, iv->nqb * 4, s));
        CK(cudaMemsetAsync(iv->thr, 0xFF, iv->nqb * 8, s));
        if (perq) {
            CK(cudaMemsetAsync(iv->surv_q, 0, iv->nqb * 8, s));
            CK(cudaMemsetAsync(iv->hash_q, 0, iv->nqb * 8, s));
        }
        if (d_probes_in)  // probes computed elsewhere (the coarse quantization split by query over ranks)
            CK(cudaMemcpyAsync(iv->probe_keys, d_probes_in, (size_t)nqb * np * 8, cudaMemcpyDeviceToDevice, s));
        else
            enumerate_cells(iv, d_q, nqb, np, s);
    }
    pb::IvfWork w{};
    w.items[0] = iv->items[0];
    w.items[1] = iv->items[1];
    w.nitems = iv->ctrl + iv->nqb + 3;
    w.cap[0] = (uint32_t)iv->items_cap[0];
    w.cap[1] = (uint32_t)iv->items_cap[1];
    w.chunk[0] = IVF_CHUNK;
    w.chunk[1] = IVF_CHUNK2;
    w.overflow = iv->ctrl + iv->nqb;
    w.lut_items[0] = iv->lut_items;
    w.lut_items[1] = iv->lut_items + (size_t)iv->nqb * np;
    w.nlut = iv->ctrl + iv->nqb + 5;
    const bool side = np > 1;
    if (phase != 2) {
    // two-phase: round 1 = the first probe exactly (>= 0 codes or 1 list reached at probe 0)
    pb::launch_ivf_probe_count(iv->probe_keys, nqb, np, iv->d_off, p->cap, iv->np_eff, iv->scanned, s, iv->split,
                               phase == 1 ? 0 : IVF_R1_CODES, phase == 1 ? 1 : IVF_R1_MAX, w);
    add_u64<<<1, 256, 0, s>>>(iv->scanned, nqb, iv->scan_total);
    pb::count_launch();
    // residual LUTs of the items with a non-empty list here: round 1's on the caller's
    // stream; round 2's on the side stream, overlapping round 1, its top-k and the
    // compaction (K1r is FP / shared-memory bound, round 1 memory / latency bound); round 2
    // waits for them
    if (side) {
        CK(cudaEventRecord(iv->ev_fork, s));
        CK(cudaStreamWaitEvent(iv->side, iv->ev_fork, 0));
        pb::launch_residual_lut(d_q, iv->dim, iv->m, iv->probe_keys, np, w.lut_items[1], w.nlut + 1, nqb * np,
                                iv->d_coarse, iv->d_codebooks, iv->d_perms, iv->lutp, iv->qcodes, iv->side);
        CK(cudaEventRecord(iv->ev_join, iv->side));
    }
    pb::launch_residual_lut(d_q, iv->dim, iv->m, iv->probe_keys, np, w.lut_items[0], w.nlut, nqb * np, iv->d_coarse,
                            iv->d_codebooks, iv->d_perms, iv->lutp, iv->qcodes, s);
    }
    pb::IvfScanArgs a{};
    a.codes = iv->d_codes_list;
    a.low = iv->d_low_list;
    a.off = iv->d_off;
    a.probe_keys = iv->probe_keys;
    a.lutp = iv->lutp;
    a.qcodes = iv->qcodes;
    a.nq = nqb;
    a.nprobe = np;
    a.tau = p->tau;
    a.thr = iv->thr;
    a.cand = iv->cand;
    a.cap = iv->cand_cap;
    a.ccount = iv->ctrl;
    a.ovq = iv->ovq;
    a.surv_total = iv->surv_total;
    // survivors are defined for the dual strategy (other strategies report 0)
    a.surv_q = perq && p->strategy == pb::DUAL ? iv->surv_q : nullptr;
    a.hash_q = perq && p->strategy == pb::DUAL ? iv->hash_q : nullptr;
    // two rounds over the work lists built by the probe-count kernel: round 1 scans each
    // query's leading probes holding >= IVF_R1_CODES codes (at most IVF_R1_MAX probes) in
    // IVF_CHUNK-row chunks; its exact k-th key (K3) bounds round 2, the remaining probes
    const uint32_t rounds = np <= 1 ? 1 : 2;  // one probe: round 1 sees everything
    // K6s: round 1's own bound from a sample of each query's first list (k <= sample)
    if (phase != 2 && IVF_SEED_ROWS && k <= IVF_SEED_ROWS / 4)
        pb::launch_ivf_seed(a, strategy, iv->m, IVF_SEED_ROWS, k, s);
    for (uint32_t round = 0; round < rounds; ++round) {
        if (phase == 1 && round == 1) break;
        if (phase == 2 && round == 0) continue;
        if (phase == 2 && d_thr) {  // the bound min-reduced over the ranks
            min_u64<<<(nqb + 255) / 256, 256, 0, s>>>(iv->thr, reinterpret_cast<const unsigned long long*>(d_thr), nqb);
            pb::count_launch();
        }
        a.items = iv->items[round];
        a.nitems = w.nitems + round;
        a.items_cap = w.cap[round];
        a.work = iv->ctrl + iv->nqb + 1 + round;
        if (round == 1 && side) CK(cudaStreamWaitEvent(s, iv->ev_join, 0));
        cudaEvent_t e1 = nullptr;
        if (iv->profiling) {
            if (iv->prof_used == iv->prof_events.size()) {
                cudaEvent_t x, y;
                CK(cudaEventCreate(&x));
                CK(cudaEventCreate(&y));
                iv->prof_events.push_back({x, y});
            }
            CK(cudaEventRecord(iv->prof_events[iv->prof_used].first, s));
            e1 = iv->prof_events[iv->prof_used++].second;
        }
        pb::launch_ivf_scan(a, strategy, iv->m, iv->num_sms, s);
        if (e1) CK(cudaEventRecord(e1, s));
        // a query whose list overflowed (in either round) is re-ranked exactly over all its
        // visited probes (no-op for the others)
        if (round + 1 == rounds) pb::launch_ivf_rescue(a, strategy, iv->m, iv->np_eff, k, s);
        pb::launch_topk(iv->cand, iv->ctrl, iv->cand_cap, 1, 0, 0, nqb, k, iv->keys, iv->kcounts, s);
        if (round == 0 && np > 1)  // bound round 2; keep only round 1's top-k as candidates
            pb::launch_seed_compact(iv->keys, iv->kcounts, nqb, k, iv->thr, iv->cand, iv->cand_cap, iv->ctrl, s);
    }
    if (phase == 1) {  // the local round-1 bound (all-ones: no bound) for the min-reduce
        CK(cudaMemcpyAsync(d_thr, iv->thr, (size_t)nqb * 8, cudaMemcpyDeviceToDevice, s));
        return;
    }
    pb::launch_or_flag(iv->sticky_overflow, iv->ctrl + iv->nqb, s);
    if (perq) {
        if (d_surv) CK(cudaMemcpyAsync(d_surv, iv->surv_q, (size_t)nqb * 8, cudaMemcpyDeviceToDevice, s));
        if (d_hash) CK(cudaMemcpyAsync(d_hash, iv->hash_q, (size_t)nqb * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (d_keys_out) {  // multi-GPU: the shard's top-k keys for the cross-rank merge
        CK(cudaMemcpyAsync(d_keys_out, iv->keys, (size_t)nqb * k * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(d_kcounts_out, iv->kcounts, nqb * 4, cudaMemcpyDeviceToDevice, s));
        return;
    }
    pb::launch_keys_to_ids(iv->keys, iv->kcounts, nqb, k, iv->idm.d_rank_to_id, d_ids, d_scores, d_counts, s);
}

// All batches; returns strategy survivors semantics (0 none, 1 = scanned, 2 counted).
int device_search(poly_b200_ivf* iv, const float* d_q, uint64_t nq, const poly_b200_ivf_params* p, int64_t* d_ids,
                  float* d_scores, uint32_t* d_counts, cudaStream_t s, uint64_t* d_keys = nullptr,
                  uint32_t* d_kcounts = nullptr, const uint64_t* d_probes = nullptr, uint64_t* d_surv = nullptr,
                  uint64_t* d_hash = nullptr) {
    validate(iv, p);
    check_pending(iv, false);
    if (nq == 0) return 0;
    if (p->k == 0 || iv->n == 0) {
        if (d_surv) CK(cudaMemsetAsync(d_surv, 0, nq * 8, s));
        if (d_hash) CK(cudaMemsetAsync(d_hash, 0, nq * 8, s));
        if (d_kcounts) {
            CK(cudaMemsetAsync(d_kcounts, 0, nq * 4, s));
            if (p->k) CK(cudaMemsetAsync(d_keys, 0xFF, nq * p->k * 8, s));
            return 0;
        }
        if (d_counts) CK(cudaMemsetAsync(d_counts, 0, nq * 4, s));
        if (p->k) pb::launch_keys_to_ids(nullptr, nullptr, (uint32_t)nq, p->k, nullptr, d_ids, d_scores, nullptr, s);
        return 0;
    }
    rebuild_lists(iv);
    ensure_ivf_scratch(iv, std::min(p->nprobe, iv->nlist), p->k);
    CK(cudaMemsetAsync(iv->surv_total, 0, 8, s));
    CK(cudaMemsetAsync(iv->scan_total, 0, 8, s));
    CK(cudaMemsetAsync(iv->sticky_overflow, 0, 4, s));
    for (uint64_t b0 = 0; b0 < nq; b0 += iv->nqb) {
        const uint32_t nqb = (uint32_t)std::min<uint64_t>(iv->nqb, nq - b0);
        const uint64_t* pr = d_probes ? d_probes + b0 * std::min(p->nprobe, iv->nlist) : nullptr;
        uint64_t* sv = d_surv ? d_surv + b0 : nullptr;
        uint64_t* hv = d_hash ? d_hash + b0 : nullptr;
        if (d_keys)
            search_batch(iv, d_q + b0 * iv->dim, nqb, p, nullptr, nullptr, nullptr, s, d_keys + b0 * p->k,
                         d_kcounts + b0, pr, sv, hv);
        else
            search_batch(iv, d_q + b0 * iv->dim, nqb, p, d_ids + b0 * p->k, d_scores + b0 * p->k,
                         d_counts ? d_counts + b0 : nullptr, s, nullptr, nullptr, pr, sv, hv);
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(iv->h_overflow, iv->sticky_overflow, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(iv->done_ev, s));
    iv->pending_check = true;
    if (p->strategy == pb::DUAL) return p->tau >= iv->code_bits() ? 1 : 2;
    return 0;
}

// Row i (id qid0 + i) of a (k+1)-NN result: drop the row's own id if present,
// else the last entry; keep at most k.
__global__ void drop_self_kernel(const int64_t* __restrict__ ids, const float* __restrict__ sc,
                                 const uint32_t* __restrict__ cnt, uint32_t nq, uint32_t k, int64_t qid0,
                                 int64_t* __restrict__ out_ids, float* __restrict__ out_sc, uint32_t* __restrict__ out_cnt) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint32_t k1 = k + 1, c = cnt[q];
    const int64_t self = qid0 + q;
    uint32_t w = 0;
    bool dropped = false;
    for (uint32_t r = 0; r < c && w < k; ++r) {
        const int64_t id = ids[(size_t)q * k1 + r];
        if (!dropped && id == self) { dropped = true; continue; }
        out_ids[(size_t)q * k + w] = id;
        out_sc[(size_t)q * k + w] = sc[(size_t)q * k1 + r];
        ++w;
    }
    for (uint32_t r = w; r < k; ++r) {
        out_ids[(size_t)q * k + r] = -1;
        out_sc[(size_t)q * k + r] = __int_as_float(0x7f800000);
    }
    if (out_cnt) out_cnt[q] = w;
}

void read_stats(poly_b200_ivf* iv, int mode, poly_b200_search_stats* st, cudaStream_t s) {
    unsigned long long h[2] = {0, 0};
    uint32_t ovf = 0;
    if (iv->scan_total) {
        CK(cudaMemcpyAsync(&h[0], iv->scan_total, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&h[1], iv->surv_total, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&ovf, iv->sticky_overflow, 4, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    iv->pending_check = false;
    *iv->h_overflow = 0;
    require(!ovf, POLY_B200_INTERNAL, "IVF work list overflow: results incomplete");
    if (st) {
        st->scanned = h[0];
        st->survivors = mode == 2 ? h[1] : (mode == 1 ? h[0] : 0);
    }
}

}  // namespace

extern "C" {

int poly_b200_ivf_create(const poly_b200_pq_desc* pq, const float* coarse, uint32_t nlist, int device,
                         poly_b200_ivf** out) {
    return guard([&] {
        require(out != nullptr, POLY_B200_INVALID_ARGUMENT, "null output handle");
        check_pq(pq);
        require(coarse != nullptr && nlist > 0, POLY_B200_INVALID_ARGUMENT, "empty coarse quantizer");
        for (uint64_t i = 0; i < (uint64_t)nlist * pq->dim; ++i)
            require(std::isfinite(coarse[i]), POLY_B200_INVALID_ARGUMENT, "non-finite coarse centroid");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, POLY_B200_INVALID_ARGUMENT, "no such CUDA device");
        DeviceGuard dg(device);
        auto* iv = new poly_b200_ivf();
        try {
            iv->device = device;
            CK(cudaDeviceGetAttribute(&iv->num_sms, cudaDevAttrMultiProcessorCount, device));
            iv->m = pq->m;
            iv->dim = (uint32_t)pq->dim;
            iv->cb = pq->m;
            iv->nlist = nlist;
            const size_t ncb = (size_t)pq->m * 256 * pb::DSUB;
            iv->h_codebooks.assign(pq->codebooks, pq->codebooks + ncb);
            iv->h_perms.assign(pq->perms, pq->perms + (size_t)pq->m * 256);
            iv->h_coarse.assign(coarse, coarse + (size_t)nlist * pq->dim);
            CK(cudaStreamCreateWithFlags(&iv->stream, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&iv->side, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&iv->ev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&iv->ev_join, cudaEventDisableTiming));
            iv->d_codebooks = dalloc<float>(ncb);
            iv->d_perms = dalloc<uint16_t>(iv->h_perms.size());
            iv->d_coarse = dalloc<float>(iv->h_coarse.size());
            iv->d_off = dalloc<uint64_t>(nlist + 1);
            CK(cudaMemcpy(iv->d_codebooks, iv->h_codebooks.data(), ncb * 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(iv->d_perms, iv->h_perms.data(), iv->h_perms.size() * 2, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(iv->d_coarse, iv->h_coarse.data(), iv->h_coarse.size() * 4, cudaMemcpyHostToDevice));
            CK(cudaMemset(iv->d_off, 0, (nlist + 1) * 8));
            // cmax >= max |c| for K5q's error bound; |c|^2 per cell comes from the pack kernel
            // (any rounding: the bound covers it)
            double cm = 0.0;
            for (uint32_t c = 0; c < nlist; ++c) {
                double acc = 0.0;
                for (size_t d = 0; d < pq->dim; ++d) {
                    const double v = iv->h_coarse[(size_t)c * pq->dim + d];
                    acc += v * v;
                }
                cm = std::max(cm, acc);
            }
            iv->cmax = (float)(std::sqrt(cm) * (1.0 + 1e-5)) + 1e-30f;
            const size_t npad = (size_t)pb::coarse_tc_tiles(nlist) * 256;
            iv->d_cnorm = dalloc<float>(npad);
            iv->d_cpacked = dalloc<float>(npad * pq->dim);
            pb::launch_coarse_pack(iv->d_coarse, nlist, (uint32_t)pq->dim, iv->d_cpacked, iv->d_cnorm, iv->stream);
            CK(cudaStreamSynchronize(iv->stream));
            CK(cudaGetLastError());
        } catch (...) {
            poly_b200_ivf_destroy(iv);
            throw;
        }
        *out = iv;
    });
}

int poly_b200_ivf_destroy(poly_b200_ivf* iv) {
    if (!iv) return POLY_B200_OK;
    return guard([&] {
        {
            DeviceGuard dg(iv->device);
            if (iv->stream) cudaStreamSynchronize(iv->stream);
            if (iv->side) cudaStreamSynchronize(iv->side);
            for (void* p : {(void*)iv->d_codebooks, (void*)iv->d_perms, (void*)iv->d_coarse, (void*)iv->d_codes_ins,
                            (void*)iv->d_cells_ins, (void*)iv->d_off, (void*)iv->d_codes_list, (void*)iv->d_low_list,
                            (void*)iv->ckeys, (void*)iv->nl_counts, (void*)iv->probe_keys, (void*)iv->probe_counts,
                            (void*)iv->np_eff, (void*)iv->split, (void*)iv->scanned, (void*)iv->lutp, (void*)iv->qcodes,
                            (void*)iv->cand, (void*)iv->ctrl, (void*)iv->thr, (void*)iv->keys, (void*)iv->kcounts,
                            (void*)iv->surv_total, (void*)iv->scan_total, (void*)iv->sticky_overflow, (void*)iv->d_q,
                            (void*)iv->ovq, (void*)iv->surv_q, (void*)iv->hash_q,
                            (void*)iv->d_oid, (void*)iv->d_osc, (void*)iv->d_ocnt,
                            (void*)iv->knn_ids, (void*)iv->knn_sc, (void*)iv->knn_cnt, (void*)iv->d_cnorm, (void*)iv->items[0],
                            (void*)iv->d_cpacked, (void*)iv->grp, (void*)iv->rank_scratch,
                            (void*)iv->items[1], (void*)iv->lut_items})
                dfree(p);
            if (iv->h_overflow) cudaFreeHost(iv->h_overflow);
            for (auto& pe : iv->prof_events) {
                cudaEventDestroy(pe.first);
                cudaEventDestroy(pe.second);
            }
            if (iv->done_ev) cudaEventDestroy(iv->done_ev);
            iv->idm.release();
            if (iv->stream) cudaStreamDestroy(iv->stream);
            if (iv->side) cudaStreamDestroy(iv->side);
            if (iv->ev_fork) cudaEventDestroy(iv->ev_fork);
            if (iv->ev_join) cudaEventDestroy(iv->ev_join);
        }
        delete iv;
    });
}

uint64_t poly_b200_ivf_size(const poly_b200_ivf* iv) { return iv ? iv->n : 0; }

int poly_b200_ivf_assign(poly_b200_ivf* iv, const float* x, uint64_t n, uint32_t* cells) {
    return guard([&] {
        require(iv && (n == 0 || (x && cells)), POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        if (n == 0) return;
        float* d_x = dalloc<float>(n * iv->dim);
        uint32_t* d_c = dalloc<uint32_t>(n);
        cudaError_t e = cudaMemcpyAsync(d_x, x, n * iv->dim * 4, cudaMemcpyHostToDevice, iv->stream);
        if (e == cudaSuccess) {
            pb::launch_assign(d_x, n, iv->dim, iv->d_coarse, iv->nlist, d_c, iv->stream);
            e = cudaMemcpyAsync(cells, d_c, n * 4, cudaMemcpyDeviceToHost, iv->stream);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(iv->stream);
        dfree(d_x);
        dfree(d_c);
        CK(e);
    });
}

int poly_b200_ivf_add_device(poly_b200_ivf* iv, const float* d_x, const uint32_t* d_cells, uint64_t n, int64_t id0,
                             void* stream) {
    return guard([&] {
        require(iv && (n == 0 || (d_x && d_cells)), POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        if (n == 0) return;
        cudaStream_t s = (cudaStream_t)stream;
        CK(cudaStreamSynchronize(s));
        grow_ins(iv, iv->n + n);
        CK(cudaMemcpyAsync(iv->d_cells_ins + iv->n, d_cells, n * 4, cudaMemcpyDeviceToDevice, iv->stream));
        pb::launch_residual_encode(d_x, n, iv->dim, iv->m, iv->d_coarse, d_cells, iv->d_codebooks, iv->d_perms,
                                   iv->d_codes_ins + iv->n * iv->cb, iv->stream);
        CK(cudaStreamSynchronize(iv->stream));
        CK(cudaGetLastError());
        iv->idm.append_range(id0, iv->n, n);
        iv->n += n;
        iv->lists_dirty = true;
    });
}

int poly_b200_ivf_add_device_ids(poly_b200_ivf* iv, const float* d_x, const uint32_t* d_cells, uint64_t n,
                                 const int64_t* ids, void* stream) {
    return guard([&] {
        require(iv && (n == 0 || (d_x && d_cells && ids)), POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        if (n == 0) return;
        cudaStream_t s = (cudaStream_t)stream;
        CK(cudaStreamSynchronize(s));
        grow_ins(iv, iv->n + n);
        CK(cudaMemcpyAsync(iv->d_cells_ins + iv->n, d_cells, n * 4, cudaMemcpyDeviceToDevice, iv->stream));
        pb::launch_residual_encode(d_x, n, iv->dim, iv->m, iv->d_coarse, d_cells, iv->d_codebooks, iv->d_perms,
                                   iv->d_codes_ins + iv->n * iv->cb, iv->stream);
        CK(cudaStreamSynchronize(iv->stream));
        CK(cudaGetLastError());
        iv->idm.append(ids, iv->n, n);
        iv->n += n;
        iv->lists_dirty = true;
    });
}

int poly_b200_ivf_add(poly_b200_ivf* iv, const float* x, uint64_t n, const uint32_t* cells, const int64_t* ids) {
    return guard([&] {
        require(iv && (n == 0 || x), POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        if (n == 0) return;
        for (uint64_t i = 0; i < n * iv->dim; ++i)
            require(std::isfinite(x[i]), POLY_B200_INVALID_ARGUMENT, "non-finite entry in vector set");
        if (cells)
            for (uint64_t i = 0; i < n; ++i) require(cells[i] < iv->nlist, POLY_B200_INVALID_ARGUMENT, "bad cell");
        grow_ins(iv, iv->n + n);
        float* d_x = dalloc<float>(n * iv->dim);
        cudaError_t e = cudaMemcpyAsync(d_x, x, n * iv->dim * 4, cudaMemcpyHostToDevice, iv->stream);
        uint32_t* d_c = iv->d_cells_ins + iv->n;
        if (e == cudaSuccess) {
            if (cells) e = cudaMemcpyAsync(d_c, cells, n * 4, cudaMemcpyHostToDevice, iv->stream);
            else pb::launch_assign(d_x, n, iv->dim, iv->d_coarse, iv->nlist, d_c, iv->stream);
        }
        if (e == cudaSuccess) {
            pb::launch_residual_encode(d_x, n, iv->dim, iv->m, iv->d_coarse, d_c, iv->d_codebooks, iv->d_perms,
                                       iv->d_codes_ins + iv->n * iv->cb, iv->stream);
            e = cudaStreamSynchronize(iv->stream);
        }
        dfree(d_x);
        CK(e);
        CK(cudaGetLastError());
        iv->idm.append(ids, iv->n, n);
        iv->n += n;
        iv->lists_dirty = true;
    });
}

int poly_b200_ivf_add_codes(poly_b200_ivf* iv, const uint32_t* cells, const uint8_t* codes, const int64_t* ids,
                            uint64_t n) {
    return guard([&] {
        require(iv && (n == 0 || (cells && codes)), POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        if (n == 0) return;
        for (uint64_t i = 0; i < n; ++i) require(cells[i] < iv->nlist, POLY_B200_INVALID_ARGUMENT, "bad cell");
        grow_ins(iv, iv->n + n);
        CK(cudaMemcpyAsync(iv->d_cells_ins + iv->n, cells, n * 4, cudaMemcpyHostToDevice, iv->stream));
        CK(cudaMemcpyAsync(iv->d_codes_ins + iv->n * iv->cb, codes, n * iv->cb, cudaMemcpyHostToDevice, iv->stream));
        CK(cudaStreamSynchronize(iv->stream));
        iv->idm.append(ids, iv->n, n);
        iv->n += n;
        iv->lists_dirty = true;
    });
}

int poly_b200_ivf_get_lists(poly_b200_ivf* iv, uint64_t* off, uint8_t* codes, int64_t* ids) {
    return guard([&] {
        require(iv != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        rebuild_lists(iv);
        if (off) std::copy(iv->h_off.begin(), iv->h_off.end(), off);
        if (codes && iv->n) CK(cudaMemcpy(codes, iv->d_codes_list, iv->n * iv->cb, cudaMemcpyDeviceToHost));
        if (ids && iv->n) {
            std::vector<uint32_t> low(iv->n);
            CK(cudaMemcpy(low.data(), iv->d_low_list, iv->n * 4, cudaMemcpyDeviceToHost));
            std::vector<int64_t> r2id;
            if (iv->idm.d_rank_to_id) {
                r2id.resize(iv->n);
                CK(cudaMemcpy(r2id.data(), iv->idm.d_rank_to_id, iv->n * 8, cudaMemcpyDeviceToHost));
            }
            for (uint64_t i = 0; i < iv->n; ++i) ids[i] = r2id.empty() ? (int64_t)low[i] : r2id[low[i]];
        }
    });
}

int poly_b200_ivf_profile_enable(poly_b200_ivf* iv, int enable) {
    return guard([&] {
        require(iv != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        std::lock_guard<std::mutex> lk(iv->mu);
        iv->profiling = enable != 0;
        iv->prof_used = 0;
    });
}

int poly_b200_ivf_profile_read(poly_b200_ivf* iv, double* scan_ms, uint64_t* scan_launches) {
    return guard([&] {
        require(iv && scan_ms && scan_launches, POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        double total = 0.0;
        for (size_t i = 0; i < iv->prof_used; ++i) {
            CK(cudaEventSynchronize(iv->prof_events[i].second));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, iv->prof_events[i].first, iv->prof_events[i].second));
            total += ms;
        }
        *scan_ms = total;
        *scan_launches = iv->prof_used;
        iv->prof_used = 0;
    });
}

// CSR of selected cells only (the CPU baseline's probed lists): off (ncells + 1),
// codes / ids in the order of `cells`.
int poly_b200_ivf_get_cells(poly_b200_ivf* iv, const uint32_t* cells, uint32_t ncells, uint64_t* off, uint8_t* codes,
                            int64_t* ids) {
    return guard([&] {
        require(iv && (ncells == 0 || (cells && off)), POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        rebuild_lists(iv);
        std::vector<int64_t> r2id;
        if (ids && iv->idm.d_rank_to_id) {
            r2id.resize(iv->n);
            CK(cudaMemcpy(r2id.data(), iv->idm.d_rank_to_id, iv->n * 8, cudaMemcpyDeviceToHost));
        }
        off[0] = 0;
        std::vector<uint32_t> low;
        for (uint32_t i = 0; i < ncells; ++i) {
            require(cells[i] < iv->nlist, POLY_B200_INVALID_ARGUMENT, "bad cell");
            const uint64_t b = iv->h_off[cells[i]], e = iv->h_off[cells[i] + 1], len = e - b;
            off[i + 1] = off[i] + len;
            if (!len) continue;
            if (codes) CK(cudaMemcpy(codes + off[i] * iv->cb, iv->d_codes_list + b * iv->cb, len * iv->cb,
                                     cudaMemcpyDeviceToHost));
            if (ids) {
                low.resize(len);
                CK(cudaMemcpy(low.data(), iv->d_low_list + b, len * 4, cudaMemcpyDeviceToHost));
                for (uint64_t j = 0; j < len; ++j) ids[off[i] + j] = r2id.empty() ? (int64_t)low[j] : r2id[low[j]];
            }
        }
    });
}

int poly_b200_ivf_set_batch(poly_b200_ivf* iv, uint32_t nqb) {
    return guard([&] {
        require(iv != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        require(nqb >= 1 && nqb <= (1u << 20), POLY_B200_INVALID_ARGUMENT, "batch must be in [1, 2^20]");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        if (nqb == iv->nqb) return;
        check_pending(iv, true);
        CK(cudaStreamSynchronize(iv->stream));
        CK(cudaStreamSynchronize(iv->side));
        CK(cudaDeviceSynchronize());  // callers' streams may still read the scratch
        // every buffer sized by the batch is reallocated lazily at the next search
        for (void** pp : {(void**)&iv->ckeys, (void**)&iv->nl_counts, (void**)&iv->grp, (void**)&iv->rank_scratch,
                          (void**)&iv->probe_keys, (void**)&iv->probe_counts, (void**)&iv->np_eff, (void**)&iv->split,
                          (void**)&iv->scanned, (void**)&iv->items[0], (void**)&iv->items[1], (void**)&iv->lutp,
                          (void**)&iv->lut_items,
                          (void**)&iv->qcodes, (void**)&iv->cand, (void**)&iv->ctrl, (void**)&iv->thr,
                          (void**)&iv->keys, (void**)&iv->kcounts, (void**)&iv->surv_total, (void**)&iv->scan_total,
                          (void**)&iv->ovq, (void**)&iv->surv_q, (void**)&iv->hash_q, (void**)&iv->sticky_overflow}) {
            dfree(*pp);
            *pp = nullptr;
        }
        if (iv->h_overflow) cudaFreeHost(iv->h_overflow);
        iv->h_overflow = nullptr;
        if (iv->done_ev) cudaEventDestroy(iv->done_ev);
        iv->done_ev = nullptr;
        iv->scratch_nprobe = 0;
        iv->items_cap[0] = iv->items_cap[1] = 0;
        iv->cand_cap = 0;
        iv->keys_k = 0;
        iv->nqb = nqb;
    });
}

uint32_t poly_b200_ivf_batch(const poly_b200_ivf* iv) { return iv ? iv->nqb : 0; }

int poly_b200_ivf_debug_set_list_capacity(poly_b200_ivf* iv, uint32_t cap) {
    return guard([&] {
        require(iv != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        std::lock_guard<std::mutex> lk(iv->mu);
        iv->cap_override = cap;
    });
}

int poly_b200_ivf_debug_rescued(poly_b200_ivf* iv, uint32_t* n) {
    return guard([&] {
        require(iv && n, POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        require(iv->ovq != nullptr, POLY_B200_STATE, "no search has run");
        CK(cudaDeviceSynchronize());
        std::vector<uint32_t> ovq(iv->nqb);
        CK(cudaMemcpy(ovq.data(), iv->ovq, iv->nqb * 4, cudaMemcpyDeviceToHost));
        *n = 0;
        for (uint32_t v : ovq) *n += v != 0;
    });
}

int poly_b200_ivf_probes(poly_b200_ivf* iv, const float* queries, uint64_t nq, uint32_t nprobe, uint32_t* cells) {
    return guard([&] {
        require(iv && (nq == 0 || (queries && cells)) && nprobe >= 1 && nprobe <= iv->nlist &&
                    nprobe <= (uint32_t)pb::KMAX,
                POLY_B200_INVALID_ARGUMENT, "bad arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        ensure_ivf_scratch(iv, nprobe, 1);
        cudaStream_t s = iv->stream;
        float* d_q = dalloc<float>(std::max<uint64_t>(nq, 1) * iv->dim);
        uint32_t* d_c = dalloc<uint32_t>((size_t)iv->nqb * nprobe);
        cudaError_t e = cudaSuccess;
        if (nq) e = cudaMemcpyAsync(d_q, queries, nq * iv->dim * 4, cudaMemcpyHostToDevice, s);
        for (uint64_t b0 = 0; b0 < nq && e == cudaSuccess; b0 += iv->nqb) {
            const uint32_t nqb = (uint32_t)std::min<uint64_t>(iv->nqb, nq - b0);
            enumerate_cells(iv, d_q + b0 * iv->dim, nqb, nprobe, s);
            probes_to_cells<<<64, 256, 0, s>>>(iv->probe_keys, (uint64_t)nqb * nprobe, d_c);
            pb::count_launch();
            e = cudaMemcpyAsync(cells + b0 * nprobe, d_c, (size_t)nqb * nprobe * 4, cudaMemcpyDeviceToHost, s);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        dfree(d_q);
        dfree(d_c);
        CK(e);
    });
}

int poly_b200_ivf_search_device_ex(poly_b200_ivf* iv, const float* d_q, uint64_t nq, const poly_b200_ivf_params* p,
                                   int64_t* d_ids, float* d_scores, uint32_t* d_counts, uint64_t* d_surv,
                                   uint64_t* d_surv_hash, void* stream, poly_b200_search_stats* stats) {
    return guard([&] {
        require(iv != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        require(nq == 0 || (d_q && d_ids && d_scores) || (p && p->k == 0), POLY_B200_INVALID_ARGUMENT, "null buffers");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        cudaStream_t s = (cudaStream_t)stream;
        const int mode =
            device_search(iv, d_q, nq, p, d_ids, d_scores, d_counts, s, nullptr, nullptr, nullptr, d_surv, d_surv_hash);
        if (stats) {
            stats->scanned = stats->survivors = 0;
            if (nq && p->k && iv->n) read_stats(iv, mode, stats, s);
        }
    });
}

int poly_b200_ivf_search_device(poly_b200_ivf* iv, const float* d_q, uint64_t nq, const poly_b200_ivf_params* p,
                                int64_t* d_ids, float* d_scores, uint32_t* d_counts, void* stream,
                                poly_b200_search_stats* stats) {
    return poly_b200_ivf_search_device_ex(iv, d_q, nq, p, d_ids, d_scores, d_counts, nullptr, nullptr, stream, stats);
}

int poly_b200_ivf_search_keys_device(poly_b200_ivf* iv, const float* d_q, uint64_t nq, const poly_b200_ivf_params* p,
                                     uint64_t* d_keys, uint32_t* d_counts, void* stream, poly_b200_search_stats* stats) {
    return guard([&] {
        require(iv != nullptr && p != nullptr, POLY_B200_INVALID_ARGUMENT, "null arguments");
        require(p->k > 0, POLY_B200_INVALID_ARGUMENT, "k must be positive for key output");
        require(nq == 0 || (d_q && d_keys && d_counts), POLY_B200_INVALID_ARGUMENT, "null buffers");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        cudaStream_t s = (cudaStream_t)stream;
        iv->idm.sync(iv->n);
        // a key carries the 32-bit low word: the id itself unless ids needed a rank table,
        // whose ranks are local to this shard and would be mis-merged across ranks
        require(iv->n == 0 || iv->idm.d_rank_to_id == nullptr, POLY_B200_STATE,
                "key output needs ids in [0, 2^32) (the key carries the id itself)");
        const int mode = device_search(iv, d_q, nq, p, nullptr, nullptr, nullptr, s, d_keys, d_counts);
        if (stats) {
            stats->scanned = stats->survivors = 0;
            if (nq && iv->n) read_stats(iv, mode, stats, s);
        }
    });
}

int poly_b200_ivf_search_keys_probes_device(poly_b200_ivf* iv, const float* d_q, uint64_t nq,
                                            const poly_b200_ivf_params* p, const uint64_t* d_probe_keys,
                                            uint64_t* d_keys, uint32_t* d_counts, void* stream,
                                            poly_b200_search_stats* stats) {
    return guard([&] {
        require(iv != nullptr && p != nullptr, POLY_B200_INVALID_ARGUMENT, "null arguments");
        require(p->k > 0, POLY_B200_INVALID_ARGUMENT, "k must be positive for key output");
        require(nq == 0 || (d_q && d_keys && d_counts && d_probe_keys), POLY_B200_INVALID_ARGUMENT, "null buffers");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        cudaStream_t s = (cudaStream_t)stream;
        iv->idm.sync(iv->n);
        // a key carries the 32-bit low word: the id itself unless ids needed a rank table,
        // whose ranks are local to this shard and would be mis-merged across ranks
        require(iv->n == 0 || iv->idm.d_rank_to_id == nullptr, POLY_B200_STATE,
                "key output needs ids in [0, 2^32) (the key carries the id itself)");
        const int mode = device_search(iv, d_q, nq, p, nullptr, nullptr, nullptr, s, d_keys, d_counts, d_probe_keys);
        if (stats) {
            stats->scanned = stats->survivors = 0;
            if (nq && iv->n) read_stats(iv, mode, stats, s);
        }
    });
}

int poly_b200_ivf_search_keys_phase_device(poly_b200_ivf* iv, const float* d_q, uint64_t nq,
                                           const poly_b200_ivf_params* p, const uint64_t* d_probe_keys, int phase,
                                           uint64_t* d_thr, uint64_t* d_keys, uint32_t* d_counts, void* stream,
                                           poly_b200_search_stats* stats) {
    return guard([&] {
        require(iv != nullptr && p != nullptr, POLY_B200_INVALID_ARGUMENT, "null arguments");
        require(phase == 1 || phase == 2, POLY_B200_INVALID_ARGUMENT, "phase must be 1 or 2");
        require(p->k > 0, POLY_B200_INVALID_ARGUMENT, "k must be positive for key output");
        require(p->cap == 0, POLY_B200_INVALID_ARGUMENT, "CoarseParams.cap > 0 is not supported with sharded lists");
        require(nq == 0 || (d_q && d_probe_keys && d_thr), POLY_B200_INVALID_ARGUMENT, "null buffers");
        require(phase == 1 || nq == 0 || (d_keys && d_counts), POLY_B200_INVALID_ARGUMENT, "null outputs");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        validate(iv, p);
        require(nq <= iv->nqb, POLY_B200_INVALID_ARGUMENT, "two-phase search takes one batch (nq <= the batch size)");
        cudaStream_t s = (cudaStream_t)stream;
        iv->idm.sync(iv->n);
        require(iv->n == 0 || iv->idm.d_rank_to_id == nullptr, POLY_B200_STATE,
                "key output needs ids in [0, 2^32) (the key carries the id itself)");
        if (phase == 1) {
            require(!iv->phase_pending, POLY_B200_STATE, "phase 1 called twice without phase 2");
            check_pending(iv, false);
            if (stats) stats->scanned = stats->survivors = 0;
            iv->phase_pending = true;
            iv->phase_nq = nq;
            iv->phase_empty = nq == 0 || iv->n == 0;
            if (iv->phase_empty) {
                if (nq) CK(cudaMemsetAsync(d_thr, 0xFF, nq * 8, s));
                return;
            }
            rebuild_lists(iv);
            ensure_ivf_scratch(iv, std::min(p->nprobe, iv->nlist), p->k);
            CK(cudaMemsetAsync(iv->surv_total, 0, 8, s));
            CK(cudaMemsetAsync(iv->scan_total, 0, 8, s));
            CK(cudaMemsetAsync(iv->sticky_overflow, 0, 4, s));
            search_batch(iv, d_q, (uint32_t)nq, p, nullptr, nullptr, nullptr, s, nullptr, nullptr, d_probe_keys, nullptr,
                         nullptr, 1, d_thr);
            CK(cudaGetLastError());
            return;
        }
        require(iv->phase_pending && iv->phase_nq == nq, POLY_B200_STATE, "phase 2 without a matching phase 1");
        iv->phase_pending = false;
        if (iv->phase_empty) {
            if (nq) {
                CK(cudaMemsetAsync(d_counts, 0, nq * 4, s));
                CK(cudaMemsetAsync(d_keys, 0xFF, nq * p->k * 8, s));
            }
            if (stats) stats->scanned = stats->survivors = 0;
            return;
        }
        search_batch(iv, d_q, (uint32_t)nq, p, nullptr, nullptr, nullptr, s, d_keys, d_counts, d_probe_keys, nullptr,
                     nullptr, 2, d_thr);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(iv->h_overflow, iv->sticky_overflow, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(iv->done_ev, s));
        iv->pending_check = true;
        if (stats) {
            stats->scanned = stats->survivors = 0;
            const int mode = p->strategy == pb::DUAL ? (p->tau >= iv->code_bits() ? 1 : 2) : 0;
            read_stats(iv, mode, stats, s);
        }
    });
}

int poly_b200_ivf_probe_keys_device(poly_b200_ivf* iv, const float* d_q, uint64_t nq, uint32_t nprobe,
                                    uint64_t* d_probe_keys, void* stream) {
    return guard([&] {
        require(iv != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        require(nprobe >= 1, POLY_B200_INVALID_ARGUMENT, "nprobe must be >= 1");
        require(std::min(nprobe, iv->nlist) <= (uint32_t)pb::KMAX, POLY_B200_INVALID_ARGUMENT,
                "min(nprobe, nlist) > 2048 is not supported on the GPU path");
        require(nq == 0 || (d_q && d_probe_keys), POLY_B200_INVALID_ARGUMENT, "null buffers");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        cudaStream_t s = (cudaStream_t)stream;
        const uint32_t np = std::min(nprobe, iv->nlist);
        if (nq == 0) return;
        rebuild_lists(iv);
        ensure_ivf_scratch(iv, np, 1);
        for (uint64_t b0 = 0; b0 < nq; b0 += iv->nqb) {
            const uint32_t nqb = (uint32_t)std::min<uint64_t>(iv->nqb, nq - b0);
            enumerate_cells(iv, d_q + b0 * iv->dim, nqb, np, s);
            CK(cudaMemcpyAsync(d_probe_keys + b0 * np, iv->probe_keys, (size_t)nqb * np * 8, cudaMemcpyDeviceToDevice,
                               s));
            CK(cudaGetLastError());
        }
    });
}

int poly_b200_ivf_merge_keys_device(poly_b200_ivf* iv, const uint64_t* d_keys, const uint32_t* d_counts,
                                    uint32_t parts, uint64_t nq, uint32_t k, int64_t* d_ids, float* d_scores,
                                    uint32_t* d_out_counts, void* stream) {
    return guard([&] {
        require(iv != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        require(parts >= 1 && parts <= 64, POLY_B200_INVALID_ARGUMENT, "parts must be in [1, 64]");
        require(k >= 1 && k <= (uint32_t)pb::KMAX, POLY_B200_INVALID_ARGUMENT, "bad k");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        cudaStream_t s = (cudaStream_t)stream;
        ensure_ivf_scratch(iv, 1, k);
        for (uint64_t b0 = 0; b0 < nq; b0 += iv->nqb) {
            const uint32_t nqb = (uint32_t)std::min<uint64_t>(iv->nqb, nq - b0);
            // parts x nq x k layout; keys carry the global id, so no id table is needed
            pb::launch_topk(reinterpret_cast<const unsigned long long*>(d_keys) + b0 * k, d_counts + b0, k, parts,
                            nq * k, nq, nqb, k, iv->keys, iv->kcounts, s);
            pb::launch_keys_to_ids(iv->keys, iv->kcounts, nqb, k, nullptr, d_ids + b0 * k, d_scores + b0 * k,
                                   d_out_counts ? d_out_counts + b0 : nullptr, s);
        }
        CK(cudaGetLastError());
    });
}

int poly_b200_ivf_knn_graph_device(poly_b200_ivf* iv, const float* d_x, uint64_t n, int64_t id0,
                                   const poly_b200_ivf_params* p, int64_t* d_ids, float* d_scores, uint32_t* d_counts,
                                   void* stream) {
    return guard([&] {
        require(iv != nullptr && p != nullptr, POLY_B200_INVALID_ARGUMENT, "null arguments");
        require(p->k >= 1 && p->k < (uint32_t)pb::KMAX, POLY_B200_INVALID_ARGUMENT, "k must be in [1, 2047]");
        require(n == 0 || (d_x && d_ids && d_scores), POLY_B200_INVALID_ARGUMENT, "null buffers");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        cudaStream_t s = (cudaStream_t)stream;
        poly_b200_ivf_params p1 = *p;
        p1.k = p->k + 1;
        const uint64_t step = 64 * iv->nqb;
        if (iv->knn_rows < std::min(step, n) || iv->knn_k1 < p1.k) {
            cudaStreamSynchronize(s);
            dfree(iv->knn_ids);
            dfree(iv->knn_sc);
            dfree(iv->knn_cnt);
            iv->knn_rows = std::max<uint64_t>(iv->knn_rows, std::min(step, n));
            iv->knn_k1 = std::max<uint32_t>(iv->knn_k1, p1.k);
            iv->knn_ids = dalloc<int64_t>(iv->knn_rows * iv->knn_k1);
            iv->knn_sc = dalloc<float>(iv->knn_rows * iv->knn_k1);
            iv->knn_cnt = dalloc<uint32_t>(iv->knn_rows);
        }
        for (uint64_t b0 = 0; b0 < n; b0 += step) {
            const uint32_t nb = (uint32_t)std::min<uint64_t>(step, n - b0);
            device_search(iv, d_x + b0 * iv->dim, nb, &p1, iv->knn_ids, iv->knn_sc, iv->knn_cnt, s);
            drop_self_kernel<<<(nb + 127) / 128, 128, 0, s>>>(iv->knn_ids, iv->knn_sc, iv->knn_cnt, nb, p->k,
                                                              id0 + (int64_t)b0, d_ids + b0 * p->k,
                                                              d_scores + b0 * p->k, d_counts ? d_counts + b0 : nullptr);
            pb::count_launch();
            read_stats(iv, 0, nullptr, s);  // syncs; fails loudly on a candidate overflow
        }
    });
}

static const char kIvfMagic[8] = {'P', 'O', 'L', 'Y', 'I', 'V', 'F', '\0'};
static const uint32_t kIvfVersion = 1;

static uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001B3ull;
    return h;
}

struct FileCloser {
    void operator()(FILE* f) const { if (f) fclose(f); }
};

// ---- k-NN graph output sink ("streamed to the output sink"; External
// Interfaces: "one record per vector -- id, neighbor count, then (neighbor id, score) pairs --
// in a sectioned binary file plus an optional ivecs export of neighbor ids").
// Layout (little-endian): magic "POLYKNNG", u32 version 1, u32 k, u64 records, then one
// section { char tag[8] = "RECORDS_", u64 bytes, u64 fnv1a64(payload), payload } whose
// payload is the records { i64 id, u32 count, count x { i64 neighbor id, f32 score } },
// packed.  The ivecs file has per record an int32 k then k int32 neighbor ids (-1 pads).
struct poly_b200_knn_writer {
    std::unique_ptr<FILE, FileCloser> f, fv;
    uint32_t k = 0;
    uint64_t records = 0, bytes = 0, hash = 0xCBF29CE484222325ull;
    // pinned double buffers for one step of rows (ids, scores, counts)
    uint64_t rows_cap = 0;
    int64_t* h_ids[2] = {nullptr, nullptr};
    float* h_sc[2] = {nullptr, nullptr};
    uint32_t* h_cnt[2] = {nullptr, nullptr};
    std::vector<uint8_t> rec;
    std::vector<int32_t> vrec;
};

namespace {
void knn_free_host(poly_b200_knn_writer* w) {
    for (int i = 0; i < 2; ++i) {
        if (w->h_ids[i]) cudaFreeHost(w->h_ids[i]);
        if (w->h_sc[i]) cudaFreeHost(w->h_sc[i]);
        if (w->h_cnt[i]) cudaFreeHost(w->h_cnt[i]);
        w->h_ids[i] = nullptr;
        w->h_sc[i] = nullptr;
        w->h_cnt[i] = nullptr;
    }
    w->rows_cap = 0;
}

void knn_put(poly_b200_knn_writer* w, FILE* f, const void* p, size_t n) {
    require(n == 0 || fwrite(p, 1, n, f) == n, POLY_B200_IO, "k-NN graph write failed");
}

// append rows [0, nb) of a host batch: ids id0 + r
void knn_write_batch(poly_b200_knn_writer* w, int slot, uint64_t nb, int64_t id0) {
    const uint32_t k = w->k;
    w->rec.clear();
    for (uint64_t r = 0; r < nb; ++r) {
        const int64_t id = id0 + (int64_t)r;
        const uint32_t c = w->h_cnt[slot][r];
        const size_t at = w->rec.size();
        w->rec.resize(at + 12 + (size_t)c * 12);
        uint8_t* o = w->rec.data() + at;
        std::memcpy(o, &id, 8);
        std::memcpy(o + 8, &c, 4);
        for (uint32_t j = 0; j < c; ++j) {
            std::memcpy(o + 12 + 12 * j, &w->h_ids[slot][r * k + j], 8);
            std::memcpy(o + 20 + 12 * j, &w->h_sc[slot][r * k + j], 4);
        }
    }
    w->hash = fnv1a(w->hash, w->rec.data(), w->rec.size());
    knn_put(w, w->f.get(), w->rec.data(), w->rec.size());
    w->bytes += w->rec.size();
    w->records += nb;
    if (w->fv) {
        w->vrec.resize((size_t)nb * (k + 1));
        for (uint64_t r = 0; r < nb; ++r) {
            int32_t* o = w->vrec.data() + r * (k + 1);
            o[0] = (int32_t)k;
            for (uint32_t j = 0; j < k; ++j)
                o[1 + j] = j < w->h_cnt[slot][r] ? (int32_t)w->h_ids[slot][r * k + j] : -1;
        }
        knn_put(w, w->fv.get(), w->vrec.data(), w->vrec.size() * 4);
    }
}
}  // namespace

int poly_b200_knn_writer_open(const char* path, const char* ivecs_path, uint32_t k, poly_b200_knn_writer** out) {
    return guard([&] {
        require(path && out, POLY_B200_INVALID_ARGUMENT, "null arguments");
        require(k >= 1 && k < (uint32_t)pb::KMAX, POLY_B200_INVALID_ARGUMENT, "k must be in [1, 2047]");
        auto w = std::make_unique<poly_b200_knn_writer>();
        w->k = k;
        w->f.reset(fopen(path, "wb"));
        require(w->f != nullptr, POLY_B200_IO, std::string("cannot open ") + path + " for writing");
        if (ivecs_path) {
            w->fv.reset(fopen(ivecs_path, "wb"));
            require(w->fv != nullptr, POLY_B200_IO, std::string("cannot open ") + ivecs_path + " for writing");
        }
        static const char magic[8] = {'P', 'O', 'L', 'Y', 'K', 'N', 'N', 'G'};
        const uint32_t ver = 1;
        const uint64_t zero = 0;
        knn_put(w.get(), w->f.get(), magic, 8);
        knn_put(w.get(), w->f.get(), &ver, 4);
        knn_put(w.get(), w->f.get(), &k, 4);
        knn_put(w.get(), w->f.get(), &zero, 8);          // records (patched at close)
        knn_put(w.get(), w->f.get(), "RECORDS_", 8);
        knn_put(w.get(), w->f.get(), &zero, 8);          // bytes (patched)
        knn_put(w.get(), w->f.get(), &zero, 8);          // checksum (patched)
        *out = w.release();
    });
}

int poly_b200_knn_writer_close(poly_b200_knn_writer* w, uint64_t* records) {
    if (!w) return POLY_B200_OK;
    std::unique_ptr<poly_b200_knn_writer> owned(w);
    return guard([&] {
        knn_free_host(w);
        FILE* f = w->f.get();
        require(fseek(f, 16, SEEK_SET) == 0, POLY_B200_IO, "k-NN graph seek failed");
        knn_put(w, f, &w->records, 8);
        require(fseek(f, 32, SEEK_SET) == 0, POLY_B200_IO, "k-NN graph seek failed");
        knn_put(w, f, &w->bytes, 8);
        knn_put(w, f, &w->hash, 8);
        require(fflush(f) == 0, POLY_B200_IO, "k-NN graph write failed");
        if (w->fv) require(fflush(w->fv.get()) == 0, POLY_B200_IO, "ivecs write failed");
        if (records) *records = w->records;
    });
}

int poly_b200_ivf_knn_graph_write_device(poly_b200_ivf* iv, poly_b200_knn_writer* w, const float* d_x, uint64_t n,
                                         int64_t id0, const poly_b200_ivf_params* p, void* stream) {
    return guard([&] {
        require(iv && w && p, POLY_B200_INVALID_ARGUMENT, "null arguments");
        require(p->k == w->k, POLY_B200_INVALID_ARGUMENT, "params.k differs from the writer's k");
        require(n == 0 || d_x, POLY_B200_INVALID_ARGUMENT, "null vectors");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        if (n == 0) return;
        cudaStream_t s = (cudaStream_t)stream;
        const uint32_t k = p->k;
        poly_b200_ivf_params p1 = *p;
        p1.k = k + 1;
        const uint64_t step = std::min<uint64_t>(64ull * iv->nqb, n);
        if (iv->knn_rows < step || iv->knn_k1 < p1.k) {
            CK(cudaStreamSynchronize(s));
            dfree(iv->knn_ids);
            dfree(iv->knn_sc);
            dfree(iv->knn_cnt);
            iv->knn_rows = std::max<uint64_t>(iv->knn_rows, step);
            iv->knn_k1 = std::max<uint32_t>(iv->knn_k1, p1.k);
            iv->knn_ids = dalloc<int64_t>(iv->knn_rows * iv->knn_k1);
            iv->knn_sc = dalloc<float>(iv->knn_rows * iv->knn_k1);
            iv->knn_cnt = dalloc<uint32_t>(iv->knn_rows);
        }
        if (w->rows_cap < step) {
            knn_free_host(w);
            for (int i = 0; i < 2; ++i) {
                CK(cudaMallocHost(&w->h_ids[i], step * k * 8));
                CK(cudaMallocHost(&w->h_sc[i], step * k * 4));
                CK(cudaMallocHost(&w->h_cnt[i], step * 4));
            }
            w->rows_cap = step;
        }
        // device outputs of one step (k per row), then copies to the pinned slot; the host
        // writes step b - 1 while the GPU searches step b
        int64_t* o_ids = dalloc<int64_t>(step * k);
        float* o_sc = dalloc<float>(step * k);
        uint32_t* o_cnt = dalloc<uint32_t>(step);
        cudaEvent_t ev[2] = {nullptr, nullptr};
        try {
            CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
            uint64_t prev_nb = 0;
            int64_t prev_id0 = 0;
            int slot = 0;
            for (uint64_t b0 = 0; b0 < n; b0 += step, slot ^= 1) {
                const uint32_t nb = (uint32_t)std::min<uint64_t>(step, n - b0);
                device_search(iv, d_x + b0 * iv->dim, nb, &p1, iv->knn_ids, iv->knn_sc, iv->knn_cnt, s);
                drop_self_kernel<<<(nb + 127) / 128, 128, 0, s>>>(iv->knn_ids, iv->knn_sc, iv->knn_cnt, nb, k,
                                                                  id0 + (int64_t)b0, o_ids, o_sc, o_cnt);
                pb::count_launch();
                CK(cudaGetLastError());
                CK(cudaMemcpyAsync(w->h_ids[slot], o_ids, (size_t)nb * k * 8, cudaMemcpyDeviceToHost, s));
                CK(cudaMemcpyAsync(w->h_sc[slot], o_sc, (size_t)nb * k * 4, cudaMemcpyDeviceToHost, s));
                CK(cudaMemcpyAsync(w->h_cnt[slot], o_cnt, (size_t)nb * 4, cudaMemcpyDeviceToHost, s));
                CK(cudaEventRecord(ev[slot], s));
                if (prev_nb) {  // the previous step's records, while this one runs
                    CK(cudaEventSynchronize(ev[slot ^ 1]));
                    knn_write_batch(w, slot ^ 1, prev_nb, prev_id0);
                }
                prev_nb = nb;
                prev_id0 = id0 + (int64_t)b0;
            }
            CK(cudaEventSynchronize(ev[slot ^ 1]));
            knn_write_batch(w, slot ^ 1, prev_nb, prev_id0);
            read_stats(iv, 0, nullptr, s);  // fails loudly on a work-list overflow
        } catch (...) {
            dfree(o_ids);
            dfree(o_sc);
            dfree(o_cnt);
            for (auto e : ev)
                if (e) cudaEventDestroy(e);
            throw;
        }
        dfree(o_ids);
        dfree(o_sc);
        dfree(o_cnt);
        for (auto e : ev) cudaEventDestroy(e);
    });
}

int poly_b200_ivf_search(poly_b200_ivf* iv, const float* queries, uint64_t nq, const poly_b200_ivf_params* p,
                         int64_t* out_ids, float* out_scores, uint32_t* out_counts, poly_b200_search_stats* stats) {
    return guard([&] {
        require(iv != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        validate(iv, p);
        require(nq == 0 || queries, POLY_B200_INVALID_ARGUMENT, "null queries");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        if (stats) *stats = {0, 0};
        if (nq == 0) return;
        const uint32_t k = std::max<uint32_t>(p->k, 1);
        cudaStream_t s = iv->stream;
        if (iv->d_q_cap < nq * iv->dim) {
            dfree(iv->d_q);
            iv->d_q_cap = nq * iv->dim;
            iv->d_q = dalloc<float>(iv->d_q_cap);
        }
        if (iv->d_out_rows < nq || iv->d_out_k < k) {
            dfree(iv->d_oid);
            dfree(iv->d_osc);
            dfree(iv->d_ocnt);
            iv->d_out_rows = std::max<uint64_t>(nq, iv->d_out_rows);
            iv->d_out_k = std::max<uint32_t>(k, iv->d_out_k);
            iv->d_oid = dalloc<int64_t>(iv->d_out_rows * iv->d_out_k);
            iv->d_osc = dalloc<float>(iv->d_out_rows * iv->d_out_k);
            iv->d_ocnt = dalloc<uint32_t>(iv->d_out_rows);
        }
        CK(cudaMemcpyAsync(iv->d_q, queries, nq * iv->dim * 4, cudaMemcpyHostToDevice, s));
        const int mode = device_search(iv, iv->d_q, nq, p, iv->d_oid, iv->d_osc, iv->d_ocnt, s);
        if (p->k) {
            CK(cudaMemcpyAsync(out_ids, iv->d_oid, nq * p->k * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(out_scores, iv->d_osc, nq * p->k * 4, cudaMemcpyDeviceToHost, s));
        }
        if (out_counts) CK(cudaMemcpyAsync(out_counts, iv->d_ocnt, nq * 4, cudaMemcpyDeviceToHost, s));
        if (p->k && iv->n) read_stats(iv, mode, stats, s);
        else CK(cudaStreamSynchronize(s));
    });
}

// ---- inverted-list file: a sectioned little-endian binary
// header { magic "POLYIVF\0", u32 version, u32 m, u32 dbits, u32 dim, u32 nlist, u32 0,
// u64 n }, then sections { char tag[8], u64 bytes, u64 fnv1a64(payload), payload } in the
// order PQCODEBK (m x 256 x dsub fp32), PQPERMS_ (m x 256 u16), COARSE__ (nlist x dim
// fp32), LISTOFF_ ((nlist + 1) u64), CODES___ (n x m u8, list order), IDS_____ (n i64).
// Errors use poly::errc (common.hpp:13-22): io, format, version, corrupt.
int poly_b200_ivf_save(poly_b200_ivf* iv, const char* path) {
    return guard([&] {
        require(iv && path, POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(iv->mu);
        DeviceGuard dg(iv->device);
        rebuild_lists(iv);
        std::unique_ptr<FILE, FileCloser> f(fopen(path, "wb"));
        require(f != nullptr, POLY_B200_IO, std::string("cannot open ") + path + " for writing");
        auto put = [&](const void* p, size_t n) {
            require(n == 0 || fwrite(p, 1, n, f.get()) == n, POLY_B200_IO, "write failed");
        };
        const uint32_t hdr[6] = {kIvfVersion, iv->m, 8u, iv->dim, iv->nlist, 0u};
        put(kIvfMagic, 8);
        put(hdr, sizeof(hdr));
        put(&iv->n, 8);
        auto section = [&](const char* tag, const void* p, uint64_t bytes) {
            const uint64_t h = fnv1a(0xCBF29CE484222325ull, p, bytes);
            put(tag, 8);
            put(&bytes, 8);
            put(&h, 8);
            put(p, bytes);
        };
        section("PQCODEBK", iv->h_codebooks.data(), iv->h_codebooks.size() * 4);
        section("PQPERMS_", iv->h_perms.data(), iv->h_perms.size() * 2);
        section("COARSE__", iv->h_coarse.data(), iv->h_coarse.size() * 4);
        section("LISTOFF_", iv->h_off.data(), iv->h_off.size() * 8);
        // codes and ids stream from the device in chunks; the checksum runs over the chunks
        const uint64_t chunk = 1ull << 24;
        std::vector<uint8_t> buf;
        auto stream_section = [&](const char* tag, uint64_t elem, auto&& fill) {
            const uint64_t bytes = iv->n * elem;
            // checksum pass first (the header precedes the payload)
            uint64_t h = 0xCBF29CE484222325ull;
            for (uint64_t i = 0; i < iv->n; i += chunk) {
                const uint64_t c = std::min(chunk, iv->n - i);
                buf.resize(c * elem);
                fill(i, c, buf.data());
                h = fnv1a(h, buf.data(), c * elem);
            }
            put(tag, 8);
            put(&bytes, 8);
            put(&h, 8);
            for (uint64_t i = 0; i < iv->n; i += chunk) {
                const uint64_t c = std::min(chunk, iv->n - i);
                buf.resize(c * elem);
                fill(i, c, buf.data());
                put(buf.data(), c * elem);
            }
        };
        stream_section("CODES___", iv->cb, [&](uint64_t i, uint64_t c, uint8_t* dst) {
            CK(cudaMemcpy(dst, iv->d_codes_list + i * iv->cb, c * iv->cb, cudaMemcpyDeviceToHost));
        });
        std::vector<int64_t> r2id;
        if (iv->idm.d_rank_to_id && iv->n) {
            r2id.resize(iv->n);
            CK(cudaMemcpy(r2id.data(), iv->idm.d_rank_to_id, iv->n * 8, cudaMemcpyDeviceToHost));
        }
        std::vector<uint32_t> low;
        stream_section("IDS_____", 8, [&](uint64_t i, uint64_t c, uint8_t* dst) {
            low.resize(c);
            CK(cudaMemcpy(low.data(), iv->d_low_list + i, c * 4, cudaMemcpyDeviceToHost));
            int64_t* o = reinterpret_cast<int64_t*>(dst);
            for (uint64_t j = 0; j < c; ++j) o[j] = r2id.empty() ? (int64_t)low[j] : r2id[low[j]];
        });
        require(fflush(f.get()) == 0, POLY_B200_IO, "write failed");
    });
}

int poly_b200_ivf_load(const char* path, int device, poly_b200_ivf** out) {
    return guard([&] {
        require(path && out, POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::unique_ptr<FILE, FileCloser> f(fopen(path, "rb"));
        require(f != nullptr, POLY_B200_IO, std::string("cannot open ") + path);
        auto get = [&](void* p, size_t n) {
            require(n == 0 || fread(p, 1, n, f.get()) == n, POLY_B200_CORRUPT, "truncated IVF list file");
        };
        char magic[8];
        uint32_t hdr[6];
        uint64_t n = 0;
        require(fread(magic, 1, 8, f.get()) == 8 && std::memcmp(magic, kIvfMagic, 8) == 0, POLY_B200_FORMAT,
                "not an IVF list file (bad magic)");
        get(hdr, sizeof(hdr));
        require(hdr[0] == kIvfVersion, POLY_B200_VERSION, "unsupported IVF list file version " + std::to_string(hdr[0]));
        get(&n, 8);
        const uint32_t m = hdr[1], dbits = hdr[2], dim = hdr[3], nlist = hdr[4];
        require(dbits == 8 && (m == 8 || m == 16) && dim == 16 * m && nlist > 0, POLY_B200_FORMAT,
                "IVF list file shape not supported on the GPU path");
        auto section = [&](const char* tag, uint64_t want, void* p) {
            char t[8];
            uint64_t bytes = 0, h = 0;
            get(t, 8);
            require(std::memcmp(t, tag, 8) == 0, POLY_B200_FORMAT, std::string("expected section ") + std::string(tag, 8));
            get(&bytes, 8);
            get(&h, 8);
            require(bytes == want, POLY_B200_FORMAT, std::string("section ") + std::string(tag, 8) + " has the wrong size");
            get(p, bytes);
            require(fnv1a(0xCBF29CE484222325ull, p, bytes) == h, POLY_B200_CORRUPT,
                    std::string("checksum mismatch in section ") + std::string(tag, 8));
        };
        std::vector<float> cb((size_t)m * 256 * pb::DSUB), coarse((size_t)nlist * dim);
        std::vector<uint16_t> perms((size_t)m * 256);
        std::vector<uint64_t> off((size_t)nlist + 1);
        section("PQCODEBK", cb.size() * 4, cb.data());
        section("PQPERMS_", perms.size() * 2, perms.data());
        section("COARSE__", coarse.size() * 4, coarse.data());
        section("LISTOFF_", off.size() * 8, off.data());
        require(off[0] == 0 && off[nlist] == n, POLY_B200_CORRUPT, "list offsets do not cover the codes");
        for (uint32_t c = 0; c < nlist; ++c) require(off[c] <= off[c + 1], POLY_B200_CORRUPT, "list offsets decrease");
        std::vector<uint8_t> codes(n * m);
        std::vector<int64_t> ids(n);
        section("CODES___", codes.size(), codes.data());
        section("IDS_____", ids.size() * 8, ids.data());
        const poly_b200_pq_desc pq{m, dbits, dim, cb.data(), perms.data()};
        poly_b200_ivf* iv = nullptr;
        int rc = poly_b200_ivf_create(&pq, coarse.data(), nlist, device, &iv);
        if (rc != POLY_B200_OK) throw Error(rc, g_err);
        std::vector<uint32_t> cells(n);
        for (uint32_t c = 0; c < nlist; ++c)
            for (uint64_t i = off[c]; i < off[c + 1]; ++i) cells[i] = c;
        rc = poly_b200_ivf_add_codes(iv, cells.data(), codes.data(), ids.data(), n);
        if (rc != POLY_B200_OK) {
            const std::string msg = g_err;
            poly_b200_ivf_destroy(iv);
            throw Error(rc, msg);
        }
        *out = iv;
    });
}

}  // extern "C"
