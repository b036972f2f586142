// capi.cu -- the C ABI declared in include/poly_b200.h.
//
// Host-side restatement of poly::FlatIndex (flat_index.hpp:99-144) over device
// memory.  The index owns device copies of the PQ tables and codes (uploaded
// once at add time), an id map, and per-batch scratch.
// Errors follow poly::errc (common.hpp:13-22) and never escape as exceptions.
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/poly_b200.h"
#include "host_common.h"
#include "poly_b200.cuh"

namespace pb {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_max_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{fn, dev}];
    if (have >= bytes) return;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess) have = bytes;
}
}  // namespace pb

namespace pbh {
thread_local std::string g_err;
}  // namespace pbh
using namespace pbh;

namespace {

constexpr uint32_t NQB = 256;  // queries per batch (BASELINE.json config 1: "batches of 256")

}  // namespace

struct poly_b200_index {
    int device = 0;
    int num_sms = 148;
    uint32_t m = 0, dbits = 0, dim = 0, cb = 0;
    std::vector<float> h_codebooks;
    std::vector<uint16_t> h_perms;
    float* d_codebooks = nullptr;
    uint16_t* d_perms = nullptr;

    // codes: n x cb bytes, capacity padded by one tile
    uint8_t* d_codes = nullptr;
    uint64_t n = 0, cap_codes = 0;

    // ids: arithmetic (id0 + pos) until a non-sequential id arrives
    pbh::IdMap idm;

    // batch scratch
    float* lutp = nullptr;
    uint8_t* qcodes = nullptr;
    unsigned long long* cand = nullptr;
    uint32_t cand_cap = 0, cand_bs = 0;
    uint32_t cap_override = 0;  // test hook: candidate-list capacity (0 = the default)
    // [ccount NQB][ovq NQB][rcount NQB][work][pad3][bdone NQB*nblk]...[group work counters (last 32)]
    uint32_t* ctrl = nullptr;
    size_t ctrl_words = 0;
    unsigned long long* thr = nullptr;
    unsigned long long* surv = nullptr;      // per-query survivors of a batch (per-query mode)
    unsigned long long* surv_hash = nullptr; // per-query survivor hashes of a batch (per-query mode)
    unsigned long long* surv_total = nullptr;  // survivors summed over the whole call
    unsigned long long* keys = nullptr;
    uint32_t keys_k = 0;
    uint32_t* kcounts = nullptr;

    // host-API staging
    float* d_q = nullptr;
    size_t d_q_cap = 0;
    int64_t* d_oid = nullptr;
    float* d_osc = nullptr;
    uint32_t* d_ocnt = nullptr;
    uint64_t d_out_rows = 0;
    uint32_t d_out_k = 0;

    cudaStream_t stream = nullptr;
    std::mutex mu;

    // K2 timing (bench.py)
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    size_t prof_used = 0;

    uint32_t code_bits() const { return m * dbits; }
};

namespace {

void grow_codes(poly_b200_index* ix, uint64_t need) {
    const uint64_t tile = pb::TILE_BYTES / ix->cb;
    if (need + tile <= ix->cap_codes) return;
    uint64_t cap = std::max<uint64_t>(need, ix->cap_codes * 2) + tile;
    cap = (cap + tile - 1) / tile * tile;
    uint8_t* p = dalloc<uint8_t>(cap * ix->cb);
    CK(cudaMemsetAsync(p, 0, cap * ix->cb, ix->stream));
    if (ix->n) CK(cudaMemcpyAsync(p, ix->d_codes, ix->n * ix->cb, cudaMemcpyDeviceToDevice, ix->stream));
    CK(cudaStreamSynchronize(ix->stream));
    dfree(ix->d_codes);
    ix->d_codes = p;
    ix->cap_codes = cap;
}

void append_ids(poly_b200_index* ix, const int64_t* ids, uint64_t n) {
    ix->idm.append(ids, ix->n, n);
}

void append_id_range(poly_b200_index* ix, int64_t first, uint64_t n) {
    ix->idm.append_range(first, ix->n, n);
}

void sync_idmap(poly_b200_index* ix) {
    ix->idm.sync(ix->n);
}

void ensure_scratch(poly_b200_index* ix, uint32_t k) {
    if (!ix->lutp) {
        ix->lutp = dalloc<float>((size_t)NQB * ix->m * 256);
        ix->qcodes = dalloc<uint8_t>((size_t)NQB * ix->cb);
        ix->thr = dalloc<unsigned long long>(NQB);
        ix->surv = dalloc<unsigned long long>(NQB);
        ix->surv_hash = dalloc<unsigned long long>(NQB);
        ix->surv_total = dalloc<unsigned long long>(1);
    }
    // select block: a block of bs list slots completes -> its k-th key tightens thr[q];
    // the list holds at least 32 * BS keys per query
    const uint32_t bs = std::max<uint32_t>(POLY_SEL_BS, POLY_SEL_KF * k);
    uint32_t cap = std::max<uint32_t>(32 * bs, 32 * pb::BS);
    if (ix->cap_override) cap = std::max<uint32_t>(2, (ix->cap_override + bs - 1) / bs) * bs;
    if (ix->cand_bs != bs || ix->cand_cap != cap) {
        dfree(ix->cand);
        dfree(ix->ctrl);
        ix->cand_bs = bs;
        ix->cand_cap = cap;
        ix->cand = dalloc<unsigned long long>((size_t)NQB * ix->cand_cap);
        ix->ctrl_words = 3 * NQB + 4 + (size_t)NQB * (cap / bs) + 32;  // + per-group work counters (last 32)
        ix->ctrl = dalloc<uint32_t>(ix->ctrl_words);
    }
    if (ix->keys_k < k) {
        dfree(ix->keys);
        dfree(ix->kcounts);
        ix->keys_k = k;
        ix->keys = dalloc<unsigned long long>((size_t)NQB * k);
        ix->kcounts = dalloc<uint32_t>(NQB);
    }
}

void validate_params(const poly_b200_index* ix, const poly_b200_search_params* p) {
    require(p != nullptr, POLY_B200_INVALID_ARGUMENT, "null search params");
    require(p->strategy >= 0 && p->strategy <= 3, POLY_B200_INVALID_ARGUMENT, "unknown strategy");
    require(p->tau <= ix->code_bits(), POLY_B200_INVALID_ARGUMENT, "tau exceeds code bits");  // SPEC.md tau in [0, M*d]
    require(p->k <= (uint32_t)pb::KMAX, POLY_B200_INVALID_ARGUMENT, "k > 2048 is not supported on the GPU path");
}

// Core batched search: per batch of <= 256 queries K1 -> K2s -> K2 (-> K2x) -> K3 into keys.
// emit(b, nqb) consumes ix->keys / ix->kcounts / ix->surv / ix->surv_hash for that batch.
// perq: per-query survivor counts and hashes in ix->surv / ix->surv_hash (else the
// exact call total accumulates in ix->surv_total at no cost in the scan).
template <class Emit>
void run_batches(poly_b200_index* ix, const float* d_queries, uint64_t nq, const poly_b200_search_params* p,
                 bool perq, cudaStream_t s, Emit&& emit) {
    const uint32_t k = p->k;
    ensure_scratch(ix, std::max<uint32_t>(k, 1));
    sync_idmap(ix);
    int strategy = p->strategy;
    const bool all_pass = strategy == pb::DUAL && p->tau >= ix->code_bits();
    if (all_pass) strategy = pb::ADC;  // dual(tau = M*d) == adc
    const uint32_t Q = (uint32_t)pb::scan_queries_per_cta(ix->m);
    const uint64_t tc = pb::TILE_BYTES / ix->cb;
    const uint64_t ntiles = (ix->n + tc - 1) / tc;
    CK(cudaMemsetAsync(ix->surv_total, 0, 8, s));
    for (uint64_t b0 = 0; b0 < nq; b0 += NQB) {
        const uint32_t nqb = (uint32_t)std::min<uint64_t>(NQB, nq - b0);
        CK(cudaMemsetAsync(ix->ctrl, 0, ix->ctrl_words * 4, s));
        CK(cudaMemsetAsync(ix->thr, 0xFF, NQB * 8, s));
        if (perq) {
            CK(cudaMemsetAsync(ix->surv, 0, NQB * 8, s));
            CK(cudaMemsetAsync(ix->surv_hash, 0, NQB * 8, s));
        }
        if (k > 0 && ix->n > 0) {
            pb::launch_lut(d_queries + b0 * ix->dim, nqb, ix->dim, ix->m, ix->d_codebooks, ix->d_perms, ix->lutp,
                           ix->qcodes, s);
            pb::ScanArgs a{};
            a.codes = ix->d_codes;
            a.n = ix->n;
            a.lutp = ix->lutp;
            a.qcodes = ix->qcodes;
            a.nqb = nqb;
            a.tau = p->tau;
            a.k = k;
            a.id_mode = ix->idm.mode;
            a.id0 = ix->idm.key_id0;
            a.id32 = ix->idm.d_id32;
            a.thr = ix->thr;
            a.ngroups = (nqb + Q - 1) / Q;
            // Seed: one CTA per query ranks a fixed 256-code-run sample (K2s).  At most
            // n / 256 runs: runs never overlap, so no code is sampled twice (a repeated
            // key would make the sample's k-th key too small and the bound invalid).
            const uint64_t seed_blocks = std::min<uint64_t>(POLY_SEED_BLOCKS, ix->n / 256);
            if (seed_blocks > 0 && ix->n > ix->cand_cap / 8)
                pb::launch_seed_sample(a, strategy, ix->m, nqb, (uint32_t)seed_blocks, s);
            a.cand = ix->cand;
            a.cap = ix->cand_cap;
            a.ccount = ix->ctrl;
            a.ovq = ix->ctrl + NQB;
            uint32_t* rcount = ix->ctrl + 2 * NQB;
            a.work = POLY_AFFINE ? ix->ctrl + ix->ctrl_words - 32 : ix->ctrl + 3 * NQB;
            a.bdone = ix->ctrl + 3 * NQB + 4;
            a.surv = perq ? ix->surv : ix->surv_total;
            a.surv_hash = perq ? ix->surv_hash : nullptr;
            const uint64_t want = std::max<uint64_t>(1, ntiles * a.ngroups / ((uint64_t)POLY_UNITS_PER_CTA * ix->num_sms));
            a.tiles_per_chunk = (uint32_t)std::min<uint64_t>(POLY_MAX_TPC, want);
            a.ntiles = ntiles;
            a.tile_stride = 1;
            a.bs = ix->cand_bs;
            a.nchunks = (uint32_t)((ntiles + a.tiles_per_chunk - 1) / a.tiles_per_chunk);
            a.units = a.nchunks * a.ngroups;
            a.affine = POLY_AFFINE;
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (ix->profiling) {
                if (ix->prof_used == ix->prof_events.size()) {
                    cudaEvent_t x, y;
                    CK(cudaEventCreate(&x));
                    CK(cudaEventCreate(&y));
                    ix->prof_events.push_back({x, y});
                }
                e0 = ix->prof_events[ix->prof_used].first;
                e1 = ix->prof_events[ix->prof_used].second;
                ++ix->prof_used;
                CK(cudaEventRecord(e0, s));
            }
            pb::launch_scan(a, strategy, ix->m, perq, ix->num_sms, s);
            if (e1) CK(cudaEventRecord(e1, s));
            CK(cudaGetLastError());
            // queries whose candidate list overflowed are re-ranked exactly (no-op otherwise)
            pb::launch_rescue(a, strategy, ix->m, rcount, ix->num_sms, s);
            pb::launch_topk(ix->cand, ix->ctrl, ix->cand_cap, 1, 0, 0, nqb, k, ix->keys, ix->kcounts, s);
        } else {
            CK(cudaMemsetAsync(ix->kcounts, 0, NQB * 4, s));
        }
        CK(cudaGetLastError());
        emit(b0, nqb, strategy == pb::DUAL, all_pass);
    }
}

__global__ void surv_out_kernel(const unsigned long long* surv, uint32_t nqb, uint64_t fill, int mode,
                                uint64_t* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nqb) out[i] = mode == 0 ? 0 : (mode == 1 ? fill : (mode == 3 ? surv[0] : surv[i]));
}

// sum over every stored code of mix64(key low word): the survivor hash when every code
// survives (dual at tau = code_bits)
__global__ void id_hash_kernel(uint64_t n, int mode, uint32_t id0, const uint32_t* __restrict__ id32,
                               unsigned long long* out) {
    unsigned long long h = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        h += pb::mix64(mode == pb::ID_ARITH ? id0 + (uint32_t)i : id32[i]);
    for (int off = 16; off; off >>= 1) h += __shfl_down_sync(0xffffffffu, h, off);
    if ((threadIdx.x & 31) == 0 && h) atomicAdd(out, h);
}

// Returns the strategy-level survivor semantics: 0 none (adc/binary/disidx),
// 1 all codes survive (dual at tau = code_bits), 2 counted by the scan.
// Per-query survivor outputs of one batch (either pointer may be null).
void emit_survivors(poly_b200_index* ix, int mode, uint32_t nqb, uint64_t* d_surv, uint64_t* d_hash, cudaStream_t s) {
    if (d_surv) {
        surv_out_kernel<<<(nqb + 127) / 128, 128, 0, s>>>(ix->surv, nqb, ix->n, mode, d_surv);
        pb::count_launch();
    }
    if (d_hash) {
        if (mode == 1) {  // every code survives: the hash of all stored ids
            CK(cudaMemsetAsync(ix->surv_hash, 0, 8, s));
            id_hash_kernel<<<4 * ix->num_sms, 256, 0, s>>>(ix->n, ix->idm.mode, ix->idm.key_id0, ix->idm.d_id32,
                                                           ix->surv_hash);
            pb::count_launch();
            surv_out_kernel<<<(nqb + 127) / 128, 128, 0, s>>>(ix->surv_hash, nqb, 0, 3, d_hash);
        } else {
            surv_out_kernel<<<(nqb + 127) / 128, 128, 0, s>>>(ix->surv_hash, nqb, 0, mode, d_hash);
        }
        pb::count_launch();
    }
}

// Returns the strategy-level survivor semantics: 0 none (adc/binary/disidx),
// 1 all codes survive (dual at tau = code_bits), 2 counted by the scan.
int device_search(poly_b200_index* ix, const float* d_queries, uint64_t nq, const poly_b200_search_params* p,
                  int64_t* d_ids, float* d_scores, uint32_t* d_counts, uint64_t* d_surv, cudaStream_t s,
                  uint64_t* d_hash = nullptr) {
    validate_params(ix, p);
    require(nq == 0 || d_queries, POLY_B200_INVALID_ARGUMENT, "null queries");
    require(p->k == 0 || (d_ids && d_scores), POLY_B200_INVALID_ARGUMENT, "null outputs");
    if (nq == 0) return 0;
    if (p->k == 0) {  // k = 0 -> empty lists
        if (d_counts) CK(cudaMemsetAsync(d_counts, 0, nq * 4, s));
        if (d_surv) CK(cudaMemsetAsync(d_surv, 0, nq * 8, s));
        if (d_hash) CK(cudaMemsetAsync(d_hash, 0, nq * 8, s));
        return 0;
    }
    const uint32_t k = p->k;
    int mode = 0;
    const bool perq = d_surv != nullptr || d_hash != nullptr;
    run_batches(ix, d_queries, nq, p, perq, s, [&](uint64_t b0, uint32_t nqb, bool dual, bool all_pass) {
        mode = dual ? 2 : (all_pass ? 1 : 0);
        pb::launch_keys_to_ids(ix->keys, ix->kcounts, nqb, k, ix->idm.d_rank_to_id, d_ids + b0 * k, d_scores + b0 * k,
                               d_counts ? d_counts + b0 : nullptr, s);
        emit_survivors(ix, mode, nqb, d_surv ? d_surv + b0 : nullptr, d_hash ? d_hash + b0 : nullptr, s);
    });
    return mode;
}

// Exact survivor total of the last device_search (syncs the stream).
uint64_t survivor_total(poly_b200_index* ix, int mode, uint64_t nq, const uint64_t* d_surv, cudaStream_t s) {
    if (mode == 0 || nq == 0) return 0;
    if (mode == 1) return ix->n * nq;
    uint64_t t = 0;
    if (d_surv) {
        std::vector<uint64_t> h(nq);
        CK(cudaMemcpyAsync(h.data(), d_surv, nq * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (uint64_t v : h) t += v;
    } else {
        CK(cudaMemcpyAsync(&t, ix->surv_total, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    return t;
}

void ensure_host_staging(poly_b200_index* ix, uint64_t nq, uint32_t k) {
    k = std::max<uint32_t>(k, 1);
    nq = std::max<uint64_t>(nq, NQB);
    if (ix->d_q_cap < nq * ix->dim) {
        dfree(ix->d_q);
        ix->d_q_cap = nq * ix->dim;
        ix->d_q = dalloc<float>(ix->d_q_cap);
    }
    if (ix->d_out_rows < nq || ix->d_out_k < k) {
        for (void* p : {(void*)ix->d_oid, (void*)ix->d_osc, (void*)ix->d_ocnt}) dfree(p);
        ix->d_out_rows = std::max<uint64_t>(nq, ix->d_out_rows);
        ix->d_out_k = std::max<uint32_t>(k, ix->d_out_k);
        ix->d_oid = dalloc<int64_t>(ix->d_out_rows * ix->d_out_k);
        ix->d_osc = dalloc<float>(ix->d_out_rows * ix->d_out_k);
        ix->d_ocnt = dalloc<uint32_t>(ix->d_out_rows);
    }
}

}  // namespace

extern "C" {

const char* poly_b200_last_error(void) { return g_err.c_str(); }

uint64_t poly_b200_launch_count(void) { return pb::g_launches.load(); }

int poly_b200_create(const poly_b200_pq_desc* pq, int device, poly_b200_index** out) {
    return guard([&] {
        require(out != nullptr, POLY_B200_INVALID_ARGUMENT, "null output handle");
        check_pq(pq);
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        require(device >= 0 && device < ndev, POLY_B200_INVALID_ARGUMENT, "no such CUDA device");
        DeviceGuard dg(device);
        auto* ix = new poly_b200_index();
        try {
            ix->device = device;
            CK(cudaDeviceGetAttribute(&ix->num_sms, cudaDevAttrMultiProcessorCount, device));
            ix->m = pq->m;
            ix->dbits = pq->dbits;
            ix->dim = (uint32_t)pq->dim;
            ix->cb = pq->m;
            const size_t ncb = (size_t)pq->m * 256 * pb::DSUB;
            ix->h_codebooks.assign(pq->codebooks, pq->codebooks + ncb);
            ix->h_perms.assign(pq->perms, pq->perms + (size_t)pq->m * 256);
            CK(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
            ix->d_codebooks = dalloc<float>(ncb);
            ix->d_perms = dalloc<uint16_t>(ix->h_perms.size());
            CK(cudaMemcpy(ix->d_codebooks, ix->h_codebooks.data(), ncb * 4, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(ix->d_perms, ix->h_perms.data(), ix->h_perms.size() * 2, cudaMemcpyHostToDevice));
            grow_codes(ix, 0);
        } catch (...) {
            poly_b200_destroy(ix);
            throw;
        }
        *out = ix;
    });
}

int poly_b200_destroy(poly_b200_index* ix) {
    if (!ix) return POLY_B200_OK;
    return guard([&] {
        {
            DeviceGuard dg(ix->device);
            if (ix->stream) cudaStreamSynchronize(ix->stream);
            for (void* p : {(void*)ix->d_codebooks, (void*)ix->d_perms, (void*)ix->d_codes, (void*)ix->lutp,
                            (void*)ix->qcodes, (void*)ix->cand, (void*)ix->ctrl, (void*)ix->thr, (void*)ix->surv,
                            (void*)ix->surv_hash, (void*)ix->surv_total, (void*)ix->keys, (void*)ix->kcounts,
                            (void*)ix->d_q, (void*)ix->d_oid, (void*)ix->d_osc, (void*)ix->d_ocnt})
                dfree(p);
            ix->idm.release();
            for (auto& pe : ix->prof_events) {
                cudaEventDestroy(pe.first);
                cudaEventDestroy(pe.second);
            }
            if (ix->stream) cudaStreamDestroy(ix->stream);
        }
        delete ix;
    });
}

uint64_t poly_b200_size(const poly_b200_index* ix) { return ix ? ix->n : 0; }
uint32_t poly_b200_code_bytes(const poly_b200_index* ix) { return ix ? ix->cb : 0; }

int poly_b200_add_codes(poly_b200_index* ix, const uint8_t* codes, const int64_t* ids, uint64_t n) {
    return guard([&] {
        require(ix != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        require(n == 0 || codes, POLY_B200_INVALID_ARGUMENT, "null codes");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        if (n == 0) return;
        grow_codes(ix, ix->n + n);
        CK(cudaMemcpyAsync(ix->d_codes + ix->n * ix->cb, codes, n * ix->cb, cudaMemcpyHostToDevice, ix->stream));
        CK(cudaStreamSynchronize(ix->stream));
        append_ids(ix, ids, n);
        ix->n += n;
    });
}

int poly_b200_add(poly_b200_index* ix, const float* x, uint64_t n, const int64_t* ids) {
    return guard([&] {
        require(ix != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        require(n == 0 || x, POLY_B200_INVALID_ARGUMENT, "null vectors");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        if (n == 0) return;  // SPEC flatindex add: n = 0 is a no-op
        for (uint64_t i = 0; i < n * ix->dim; ++i)
            require(std::isfinite(x[i]), POLY_B200_INVALID_ARGUMENT, "non-finite entry in vector set");
        grow_codes(ix, ix->n + n);
        const uint64_t step = 1 << 20;
        float* d_x = dalloc<float>(std::min(n, step) * ix->dim);
        try {
            for (uint64_t b = 0; b < n; b += step) {
                const uint64_t c = std::min(step, n - b);
                CK(cudaMemcpyAsync(d_x, x + b * ix->dim, c * ix->dim * 4, cudaMemcpyHostToDevice, ix->stream));
                pb::launch_encode(d_x, c, ix->dim, ix->m, ix->d_codebooks, ix->d_perms,
                                  ix->d_codes + (ix->n + b) * ix->cb, ix->stream);
                CK(cudaGetLastError());
            }
            CK(cudaStreamSynchronize(ix->stream));
        } catch (...) {
            dfree(d_x);
            throw;
        }
        dfree(d_x);
        append_ids(ix, ids, n);
        ix->n += n;
    });
}

int poly_b200_add_synthetic(poly_b200_index* ix, uint64_t seed, const float* centers, uint32_t ncent,
                            uint32_t stream_id, uint64_t row0, uint64_t n, int normalize) {
    return guard([&] {
        require(ix && centers && ncent > 0, POLY_B200_INVALID_ARGUMENT, "bad synthetic arguments");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        if (n == 0) return;
        grow_codes(ix, ix->n + n);
        float* d_c = dalloc<float>((size_t)ncent * ix->dim);
        CK(cudaMemcpy(d_c, centers, (size_t)ncent * ix->dim * 4, cudaMemcpyHostToDevice));
        pb::launch_synth_encode(seed, stream_id, row0, n, d_c, ncent, ix->dim, normalize, ix->m, ix->d_codebooks,
                                ix->d_perms, ix->d_codes + ix->n * ix->cb, ix->stream);
        cudaError_t e = cudaStreamSynchronize(ix->stream);
        dfree(d_c);
        CK(e);
        CK(cudaGetLastError());
        append_id_range(ix, (int64_t)row0, n);
        ix->n += n;
    });
}

int poly_b200_gen_points_device(int device, uint64_t seed, const float* centers, uint32_t ncent, uint32_t dim,
                                uint32_t stream_id, uint64_t row0, uint64_t n, int normalize, float* d_out,
                                void* stream) {
    return guard([&] {
        require(centers && d_out, POLY_B200_INVALID_ARGUMENT, "null buffers");
        DeviceGuard dg(device);
        float* d_c = dalloc<float>((size_t)ncent * dim);
        CK(cudaMemcpy(d_c, centers, (size_t)ncent * dim * 4, cudaMemcpyHostToDevice));
        pb::launch_gen_points(seed, stream_id, row0, n, d_c, ncent, dim, normalize, d_out, (cudaStream_t)stream);
        cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
        dfree(d_c);
        CK(e);
    });
}

int poly_b200_search_batch_device_ex(poly_b200_index* ix, const float* d_queries, uint64_t nq,
                                     const poly_b200_search_params* p, int64_t* d_ids, float* d_scores,
                                     uint32_t* d_counts, uint64_t* d_surv, uint64_t* d_surv_hash, void* stream,
                                     poly_b200_search_stats* stats) {
    return guard([&] {
        require(ix != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        cudaStream_t s = (cudaStream_t)stream;
        const int mode = device_search(ix, d_queries, nq, p, d_ids, d_scores, d_counts, d_surv, s, d_surv_hash);
        if (stats) {
            stats->scanned = ix->n * nq;
            stats->survivors = survivor_total(ix, mode, nq, d_surv, s);
        }
    });
}

int poly_b200_search_batch_device(poly_b200_index* ix, const float* d_queries, uint64_t nq,
                                  const poly_b200_search_params* p, int64_t* d_ids, float* d_scores,
                                  uint32_t* d_counts, uint64_t* d_surv, void* stream, poly_b200_search_stats* stats) {
    return poly_b200_search_batch_device_ex(ix, d_queries, nq, p, d_ids, d_scores, d_counts, d_surv, nullptr, stream,
                                            stats);
}

int poly_b200_search_batch(poly_b200_index* ix, const float* queries, uint64_t nq, const poly_b200_search_params* p,
                           int64_t* out_ids, float* out_scores, uint32_t* out_counts, poly_b200_search_stats* stats) {
    return guard([&] {
        require(ix != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        validate_params(ix, p);
        require(nq == 0 || queries, POLY_B200_INVALID_ARGUMENT, "null queries");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        if (stats) *stats = {ix->n * nq, 0};
        if (nq == 0) return;
        const uint32_t k = p->k;
        ensure_host_staging(ix, nq, k);
        cudaStream_t s = ix->stream;
        CK(cudaMemcpyAsync(ix->d_q, queries, nq * ix->dim * 4, cudaMemcpyHostToDevice, s));
        const int mode = device_search(ix, ix->d_q, nq, p, ix->d_oid, ix->d_osc, ix->d_ocnt, nullptr, s);
        if (k) {
            CK(cudaMemcpyAsync(out_ids, ix->d_oid, nq * k * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(out_scores, ix->d_osc, nq * k * 4, cudaMemcpyDeviceToHost, s));
        }
        if (out_counts) CK(cudaMemcpyAsync(out_counts, ix->d_ocnt, nq * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (stats) stats->survivors = survivor_total(ix, mode, nq, nullptr, s);
    });
}

int poly_b200_search_keys_device(poly_b200_index* ix, const float* d_queries, uint64_t nq,
                                 const poly_b200_search_params* p, uint64_t* d_keys, uint32_t* d_counts,
                                 uint64_t* d_surv, void* stream) {
    return guard([&] {
        require(ix != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        validate_params(ix, p);
        require(p->k > 0, POLY_B200_INVALID_ARGUMENT, "k must be positive for key output");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        cudaStream_t s = (cudaStream_t)stream;
        sync_idmap(ix);
        // a key carries the 32-bit low word: the id itself unless ids needed a rank table,
        // whose ranks are local to this shard and would be mis-merged across ranks
        require(ix->n == 0 || ix->idm.d_rank_to_id == nullptr, POLY_B200_STATE,
                "key output needs ids in [0, 2^32) (the key carries the id itself)");
        const uint32_t k = p->k;
        run_batches(ix, d_queries, nq, p, d_surv != nullptr, s, [&](uint64_t b0, uint32_t nqb, bool dual, bool all_pass) {
            CK(cudaMemcpyAsync(d_keys + b0 * k, ix->keys, (size_t)nqb * k * 8, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(d_counts + b0, ix->kcounts, nqb * 4, cudaMemcpyDeviceToDevice, s));
            emit_survivors(ix, dual ? 2 : (all_pass ? 1 : 0), nqb, d_surv ? d_surv + b0 : nullptr, nullptr, s);
        });
    });
}

int poly_b200_merge_keys_device(poly_b200_index* ix, const uint64_t* d_keys, const uint32_t* d_counts, uint32_t parts,
                                uint64_t nq, uint32_t k, int64_t* d_ids, float* d_scores, uint32_t* d_out_counts,
                                void* stream) {
    return guard([&] {
        require(ix != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        require(parts >= 1 && parts <= 64, POLY_B200_INVALID_ARGUMENT, "parts must be in [1, 64]");
        require(k >= 1 && k <= (uint32_t)pb::KMAX, POLY_B200_INVALID_ARGUMENT, "bad k");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        cudaStream_t s = (cudaStream_t)stream;
        ensure_scratch(ix, k);
        sync_idmap(ix);
        for (uint64_t b0 = 0; b0 < nq; b0 += NQB) {
            const uint32_t nqb = (uint32_t)std::min<uint64_t>(NQB, nq - b0);
            // parts x nq x k layout: part p of batch query i at d_keys + (p * nq + b0 + i) * k
            pb::launch_topk(reinterpret_cast<const unsigned long long*>(d_keys) + b0 * k, d_counts + b0, k, parts,
                            nq * k, nq, nqb, k, ix->keys, ix->kcounts, s);
            pb::launch_keys_to_ids(ix->keys, ix->kcounts, nqb, k, ix->idm.d_rank_to_id, d_ids + b0 * k, d_scores + b0 * k,
                                   d_out_counts ? d_out_counts + b0 : nullptr, s);
        }
        CK(cudaGetLastError());
    });
}

int poly_b200_calibrate_threshold(poly_b200_index* ix, const float* train_queries, uint64_t nq, double rate,
                                  uint32_t* tau, int* warning) {
    return guard([&] {
        require(ix && tau, POLY_B200_INVALID_ARGUMENT, "null arguments");
        require(rate > 0.0 && rate < 1.0, POLY_B200_INVALID_ARGUMENT, "target filter rate must be in (0, 1)");
        require(nq == 0 || train_queries, POLY_B200_INVALID_ARGUMENT, "null queries");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        ensure_scratch(ix, 1);
        ensure_host_staging(ix, nq, 1);
        cudaStream_t s = ix->stream;
        const uint32_t nb = ix->code_bits() + 1;
        unsigned long long* d_hist = dalloc<unsigned long long>(std::max<uint64_t>(nq, 1) * nb);
        std::vector<unsigned long long> hist(nq * nb);
        try {
            CK(cudaMemsetAsync(d_hist, 0, std::max<uint64_t>(nq, 1) * nb * 8, s));
            if (nq) CK(cudaMemcpyAsync(ix->d_q, train_queries, nq * ix->dim * 4, cudaMemcpyHostToDevice, s));
            for (uint64_t b0 = 0; b0 < nq; b0 += NQB) {
                const uint32_t nqb = (uint32_t)std::min<uint64_t>(NQB, nq - b0);
                pb::launch_lut(ix->d_q + b0 * ix->dim, nqb, ix->dim, ix->m, ix->d_codebooks, ix->d_perms, ix->lutp,
                               ix->qcodes, s);
                pb::launch_hamming_hist(ix->d_codes, ix->n, ix->cb, ix->qcodes, nqb, d_hist + b0 * nb, s);
            }
            if (nq) CK(cudaMemcpyAsync(hist.data(), d_hist, nq * nb * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        } catch (...) {
            dfree(d_hist);
            throw;
        }
        dfree(d_hist);
        // max { tau : mean survivor fraction <= 1 - rate } (flat_index.hpp:128-130)
        if (warning) *warning = 0;
        double cum = 0.0;
        int64_t best = -1;
        for (uint32_t t = 0; t < nb; ++t) {
            for (uint64_t i = 0; i < nq; ++i) cum += (double)hist[i * nb + t];
            const double frac = (nq && ix->n) ? cum / ((double)nq * (double)ix->n) : 0.0;
            if (frac <= 1.0 - rate) best = t;
        }
        if (best < 0) {
            if (warning) *warning = 1;
            *tau = 0;
        } else {
            *tau = (uint32_t)best;
        }
    });
}

int poly_b200_with_assignments(const poly_b200_index* src, const uint16_t* perms, poly_b200_index** out) {
    return guard([&] {
        require(src && perms && out, POLY_B200_INVALID_ARGUMENT, "null arguments");
        poly_b200_pq_desc d{src->m, src->dbits, src->dim, src->h_codebooks.data(), perms};
        poly_b200_index* dst = nullptr;
        const int rc = poly_b200_create(&d, src->device, &dst);
        if (rc != POLY_B200_OK) throw Error(rc, g_err);
        try {
            DeviceGuard dg(src->device);
            grow_codes(dst, src->n);
            // field f -> new_perm[old_inv_perm[f]] per sub-quantizer
            std::vector<uint8_t> maps((size_t)src->m * 256);
            for (uint32_t sq = 0; sq < src->m; ++sq) {
                std::vector<uint16_t> inv(256);
                for (uint32_t j = 0; j < 256; ++j) inv[src->h_perms[sq * 256 + j]] = (uint16_t)j;
                for (uint32_t f = 0; f < 256; ++f) maps[sq * 256 + f] = (uint8_t)perms[sq * 256 + inv[f]];
            }
            uint8_t* d_maps = dalloc<uint8_t>(maps.size());
            CK(cudaMemcpy(d_maps, maps.data(), maps.size(), cudaMemcpyHostToDevice));
            if (src->n) {
                CK(cudaMemcpyAsync(dst->d_codes, src->d_codes, src->n * src->cb, cudaMemcpyDeviceToDevice, dst->stream));
                pb::launch_relabel(dst->d_codes, src->n, src->m, d_maps, dst->stream);
            }
            cudaError_t e = cudaStreamSynchronize(dst->stream);
            dfree(d_maps);
            CK(e);
            dst->n = src->n;
            dst->idm.arith = src->idm.arith;
            dst->idm.id0 = src->idm.id0;
            dst->idm.h = src->idm.h;
            dst->idm.dirty = true;
        } catch (...) {
            poly_b200_destroy(dst);
            throw;
        }
        *out = dst;
    });
}

int poly_b200_debug_lut(poly_b200_index* ix, const float* queries, uint64_t nq, float* lutp, uint8_t* qcodes) {
    return guard([&] {
        require(ix && queries && lutp && qcodes, POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        ensure_scratch(ix, 1);
        ensure_host_staging(ix, nq, 1);
        cudaStream_t s = ix->stream;
        CK(cudaMemcpyAsync(ix->d_q, queries, nq * ix->dim * 4, cudaMemcpyHostToDevice, s));
        for (uint64_t b0 = 0; b0 < nq; b0 += NQB) {
            const uint32_t nqb = (uint32_t)std::min<uint64_t>(NQB, nq - b0);
            pb::launch_lut(ix->d_q + b0 * ix->dim, nqb, ix->dim, ix->m, ix->d_codebooks, ix->d_perms, ix->lutp,
                           ix->qcodes, s);
            CK(cudaMemcpyAsync(lutp + b0 * ix->m * 256, ix->lutp, (size_t)nqb * ix->m * 256 * 4,
                               cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(qcodes + b0 * ix->cb, ix->qcodes, (size_t)nqb * ix->cb, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
    });
}

int poly_b200_debug_set_list_capacity(poly_b200_index* ix, uint32_t cap) {
    return guard([&] {
        require(ix != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        ix->cap_override = cap;
    });
}

int poly_b200_debug_rescued(poly_b200_index* ix, uint32_t* n) {
    return guard([&] {
        require(ix && n, POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        require(ix->ctrl != nullptr, POLY_B200_STATE, "no search has run");
        CK(cudaDeviceSynchronize());
        std::vector<uint32_t> ovq(NQB);
        CK(cudaMemcpy(ovq.data(), ix->ctrl + NQB, NQB * 4, cudaMemcpyDeviceToHost));
        *n = 0;
        for (uint32_t v : ovq) *n += v != 0;
    });
}

int poly_b200_debug_counts(poly_b200_index* ix, uint32_t* ccount, uint64_t* thr, uint32_t nq) {
    return guard([&] {
        require(ix && ccount && thr && nq <= NQB, POLY_B200_INVALID_ARGUMENT, "bad arguments");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        require(ix->ctrl != nullptr, POLY_B200_STATE, "no search has run");
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(ccount, ix->ctrl, nq * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(thr, ix->thr, nq * 8, cudaMemcpyDeviceToHost));
    });
}

int poly_b200_profile_enable(poly_b200_index* ix, int enable) {
    return guard([&] {
        require(ix != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        ix->profiling = enable != 0;
        ix->prof_used = 0;
    });
}

int poly_b200_profile_read(poly_b200_index* ix, double* scan_ms, uint64_t* scan_launches) {
    return guard([&] {
        require(ix && scan_ms && scan_launches, POLY_B200_INVALID_ARGUMENT, "null arguments");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        double total = 0.0;
        for (size_t i = 0; i < ix->prof_used; ++i) {
            CK(cudaEventSynchronize(ix->prof_events[i].second));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ix->prof_events[i].first, ix->prof_events[i].second));
            total += ms;
        }
        *scan_ms = total;
        *scan_launches = ix->prof_used;
        ix->prof_used = 0;
    });
}

int poly_b200_get_codes(const poly_b200_index* ix, uint8_t* codes, int64_t* ids) {
    return guard([&] {
        require(ix != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        DeviceGuard dg(ix->device);
        if (codes && ix->n) CK(cudaMemcpy(codes, ix->d_codes, ix->n * ix->cb, cudaMemcpyDeviceToHost));
        if (ids)
            for (uint64_t i = 0; i < ix->n; ++i) ids[i] = ix->idm.at(i);
    });
}

}  // extern "C"
