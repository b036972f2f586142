// capi_multi.cu -- one FlatIndex over several GPUs of one process (include/poly_b200.h,
// poly_b200_sharded_*): SURVEY.md sec. 8(b)/(e) `create(pq_desc, n_gpus, ...)`.
//
// The database is partitioned by insertion order: every add / add_codes call
// splits its rows into n contiguous parts, part g to the shard on devices[g],
// each row keeping its global id (FlatIndex ids, flat_index.hpp:40).  A search
// runs the single-device path (K1 -> K2s -> K2 -> K3) on every shard
// concurrently, one host thread per shard, each on its own device and stream;
// the per-shard top-k lists (ascending (score, id)) are merged on
// the first device by K3g, which reads them in place over peer memory (NVLink on
// a B200 node): gather and merge in one kernel, exact for arbitrary int64 ids
// since the shards hold disjoint rows (peer copies + K3m, an n-way merge per
// query, when a device cannot load from a peer or k is large).  This is the
// single-process counterpart of distributed.ShardedSearch (one rank per GPU,
// NCCL all-gather); both merge the same lists.
#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/poly_b200.h"
#include "host_common.h"
#include "poly_b200.cuh"

using namespace pbh;

namespace pb {

// K3m: per query, merge `parts` sorted top-k lists (ids / scores parts x nq x k,
// counts parts x nq; a list holds counts[p][q] entries) into the first k entries
// of their union in (score, id) order.  One thread per query: k x parts steps.
__global__ void merge_sorted_kernel(const int64_t* __restrict__ ids, const float* __restrict__ sc,
                                    const uint32_t* __restrict__ cnt, uint32_t parts, uint32_t nq, uint32_t k,
                                    int64_t* __restrict__ out_ids, float* __restrict__ out_sc,
                                    uint32_t* __restrict__ out_cnt) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    constexpr uint32_t PMAX = 64;
    uint32_t head[PMAX];
    for (uint32_t p = 0; p < parts; ++p) head[p] = 0;
    uint32_t w = 0;
    for (; w < k; ++w) {
        int best = -1;
        float bs = 0.f;
        int64_t bi = 0;
        for (uint32_t p = 0; p < parts; ++p) {
            const size_t row = ((size_t)p * nq + q);
            if (head[p] >= cnt[row]) continue;
            const float s = sc[row * k + head[p]];
            const int64_t id = ids[row * k + head[p]];
            if (best < 0 || s < bs || (s == bs && id < bi)) {
                best = (int)p;
                bs = s;
                bi = id;
            }
        }
        if (best < 0) break;
        ++head[best];
        out_ids[(size_t)q * k + w] = bi;
        out_sc[(size_t)q * k + w] = bs;
    }
    if (out_cnt) out_cnt[q] = w;
    for (uint32_t r = w; r < k; ++r) {
        out_ids[(size_t)q * k + r] = -1;
        out_sc[(size_t)q * k + r] = __int_as_float(0x7f800000);
    }
}

// K3g: gather + merge in one kernel.  The shards' top-k lists are read where they lie -- on the
// shards' own devices, through peer memory (NVLink P2P loads; plain loads for a shard on this
// device) -- so there is no copy step between the shard searches and the merge.  One warp per
// query: coalesced loads stage the query's `parts` sorted lists in shared memory, then every
// entry finds its rank in the union by binary searches in the other lists ((score, id) order:
// ids are distinct across shards, so the ranks are a permutation) and the entries of rank < k
// are written out.
constexpr uint32_t GM_PARTS = 64, GM_WARPS = 4;
struct GatherSrc {
    const int64_t* ids[GM_PARTS];
    const float* sc[GM_PARTS];
    const uint32_t* cnt[GM_PARTS];
};

__device__ __forceinline__ bool gm_less(float s, int64_t id, float s2, int64_t id2) {
    return s < s2 || (s == s2 && id < id2);
}

__global__ void __launch_bounds__(GM_WARPS * 32) gather_merge_kernel(const GatherSrc src, uint32_t parts, uint32_t nq,
                                                                      uint32_t k, int64_t* __restrict__ out_ids,
                                                                      float* __restrict__ out_sc,
                                                                      uint32_t* __restrict__ out_cnt) {
    extern __shared__ __align__(16) uint8_t gm_smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q = blockIdx.x * GM_WARPS + warp;
    if (q >= nq) return;  // warps are independent: no CTA barrier below
    const size_t per_warp = (((size_t)parts * k * 12 + 15) & ~(size_t)15) + (size_t)GM_PARTS * 4;  // as the host sizes it
    int64_t* s_id = reinterpret_cast<int64_t*>(gm_smem + warp * per_warp);
    float* s_sc = reinterpret_cast<float*>(s_id + (size_t)parts * k);
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(gm_smem + warp * per_warp + (((size_t)parts * k * 12 + 15) & ~(size_t)15));
    for (uint32_t p = lane; p < parts; p += 32) s_cnt[p] = min(src.cnt[p][q], k);
    __syncwarp();
    uint32_t total = 0;
    for (uint32_t p = 0; p < parts; ++p) {
        const uint32_t c = s_cnt[p];
        total += c;
        const int64_t* gi = src.ids[p] + (size_t)q * k;
        const float* gs = src.sc[p] + (size_t)q * k;
        for (uint32_t i = lane; i < c; i += 32) {
            s_id[p * k + i] = gi[i];
            s_sc[p * k + i] = gs[i];
        }
    }
    __syncwarp();
    for (uint32_t p = 0; p < parts; ++p) {
        const uint32_t c = s_cnt[p];
        for (uint32_t i = lane; i < c; i += 32) {
            const float s = s_sc[p * k + i];
            const int64_t id = s_id[p * k + i];
            uint32_t rank = i;
            for (uint32_t p2 = 0; p2 < parts && rank < k; ++p2) {
                if (p2 == p) continue;
                uint32_t lo = 0, hi = s_cnt[p2];  // entries of list p2 before (s, id)
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (gm_less(s_sc[p2 * k + mid], s_id[p2 * k + mid], s, id)) lo = mid + 1;
                    else hi = mid;
                }
                rank += lo;
            }
            if (rank < k) {
                out_ids[(size_t)q * k + rank] = id;
                out_sc[(size_t)q * k + rank] = s;
            }
        }
    }
    const uint32_t w = min(total, k);
    if (lane == 0 && out_cnt) out_cnt[q] = w;
    for (uint32_t r = w + lane; r < k; r += 32) {
        out_ids[(size_t)q * k + r] = -1;
        out_sc[(size_t)q * k + r] = __int_as_float(0x7f800000);
    }
}

}  // namespace pb

struct poly_b200_sharded {
    std::vector<int> devices;
    std::vector<poly_b200_index*> shards;
    std::vector<char> direct;  // shard g's buffers are loadable from devices[0] (same device or peer access enabled)
    uint32_t m = 0, dim = 0, cb = 0, code_bits = 0;
    uint64_t n = 0;
    // per-shard device staging (queries in, top-k out) on the shard's device
    struct Stage {
        float* d_q = nullptr;
        int64_t* d_ids = nullptr;
        float* d_sc = nullptr;
        uint32_t* d_cnt = nullptr;
        cudaStream_t stream = nullptr;
        cudaEvent_t done = nullptr;
    };
    std::vector<Stage> st;
    uint64_t st_rows = 0;
    uint32_t st_k = 0;
    // gather + merge on devices[0]
    int64_t* g_ids = nullptr;
    float* g_sc = nullptr;
    uint32_t* g_cnt = nullptr;
    int64_t* o_ids = nullptr;
    float* o_sc = nullptr;
    uint32_t* o_cnt = nullptr;
    std::mutex mu;
};

namespace {

void free_staging(poly_b200_sharded* h) {
    for (size_t g = 0; g < h->st.size(); ++g) {
        DeviceGuard dg(h->devices[g]);
        auto& s = h->st[g];
        if (s.stream) cudaStreamSynchronize(s.stream);
        dfree(s.d_q);
        dfree(s.d_ids);
        dfree(s.d_sc);
        dfree(s.d_cnt);
        s.d_q = nullptr;
        s.d_ids = nullptr;
        s.d_sc = nullptr;
        s.d_cnt = nullptr;
    }
    if (!h->devices.empty()) {
        DeviceGuard dg(h->devices[0]);
        for (void* p : {(void*)h->g_ids, (void*)h->g_sc, (void*)h->g_cnt, (void*)h->o_ids, (void*)h->o_sc,
                        (void*)h->o_cnt})
            dfree(p);
    }
    h->g_ids = nullptr;
    h->g_sc = nullptr;
    h->g_cnt = nullptr;
    h->o_ids = nullptr;
    h->o_sc = nullptr;
    h->o_cnt = nullptr;
    h->st_rows = 0;
    h->st_k = 0;
}

void ensure_staging(poly_b200_sharded* h, uint64_t nq, uint32_t k) {
    if (nq <= h->st_rows && k <= h->st_k) return;
    free_staging(h);
    const uint64_t rows = std::max<uint64_t>(nq, 1);
    const uint32_t kk = std::max<uint32_t>(k, 1);
    const size_t P = h->shards.size();
    for (size_t g = 0; g < P; ++g) {
        DeviceGuard dg(h->devices[g]);
        auto& s = h->st[g];
        s.d_q = dalloc<float>(rows * h->dim);
        s.d_ids = dalloc<int64_t>(rows * kk);
        s.d_sc = dalloc<float>(rows * kk);
        s.d_cnt = dalloc<uint32_t>(rows);
    }
    DeviceGuard dg(h->devices[0]);
    h->g_ids = dalloc<int64_t>(P * rows * kk);
    h->g_sc = dalloc<float>(P * rows * kk);
    h->g_cnt = dalloc<uint32_t>(P * rows);
    h->o_ids = dalloc<int64_t>(rows * kk);
    h->o_sc = dalloc<float>(rows * kk);
    h->o_cnt = dalloc<uint32_t>(rows);
    h->st_rows = rows;
    h->st_k = kk;
}

void rethrow(int rc) {
    if (rc != POLY_B200_OK) throw Error(rc, g_err);
}

// run f(g) for every shard, one thread per shard; the first failure is rethrown
template <class F>
void for_shards(poly_b200_sharded* h, F&& f) {
    const size_t P = h->shards.size();
    std::vector<int> rc(P, POLY_B200_OK);
    std::vector<std::string> msg(P);
    auto body = [&](size_t g) {
        rc[g] = guard([&] { f(g); });
        if (rc[g] != POLY_B200_OK) msg[g] = g_err;
    };
    if (P == 1) {
        body(0);
    } else {
        std::vector<std::thread> th;
        th.reserve(P);
        for (size_t g = 0; g < P; ++g) th.emplace_back(body, g);
        for (auto& t : th) t.join();
    }
    for (size_t g = 0; g < P; ++g)
        if (rc[g] != POLY_B200_OK) throw Error(rc[g], "shard " + std::to_string(g) + ": " + msg[g]);
}

// rows [g n / P, (g + 1) n / P) of an add call go to shard g
uint64_t part_lo(uint64_t n, size_t P, size_t g) { return (uint64_t)((__uint128_t)n * g / P); }

}  // namespace

extern "C" {

int poly_b200_sharded_create(const poly_b200_pq_desc* pq, const int* devices, uint32_t n_devices,
                             poly_b200_sharded** out) {
    return guard([&] {
        require(out != nullptr && devices != nullptr, POLY_B200_INVALID_ARGUMENT, "null arguments");
        require(n_devices >= 1 && n_devices <= 64, POLY_B200_INVALID_ARGUMENT, "n_devices must be in [1, 64]");
        auto h = std::make_unique<poly_b200_sharded>();
        h->devices.assign(devices, devices + n_devices);
        h->st.resize(n_devices);
        try {
            for (uint32_t g = 0; g < n_devices; ++g) {
                poly_b200_index* ix = nullptr;
                rethrow(poly_b200_create(pq, devices[g], &ix));
                h->shards.push_back(ix);
                DeviceGuard dg(devices[g]);
                CK(cudaStreamCreateWithFlags(&h->st[g].stream, cudaStreamNonBlocking));
                CK(cudaEventCreateWithFlags(&h->st[g].done, cudaEventDisableTiming));
            }
            // peer access lets K3g load the shards' lists from devices[0] over NVLink
            h->direct.assign(n_devices, 1);
            for (uint32_t g = 1; g < n_devices; ++g) {
                if (devices[g] == devices[0]) continue;
                int can = 0;
                CK(cudaDeviceCanAccessPeer(&can, devices[0], devices[g]));
                if (can) {
                    DeviceGuard dg(devices[0]);
                    const cudaError_t e = cudaDeviceEnablePeerAccess(devices[g], 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else CK(e);
                }
                h->direct[g] = (char)(can != 0);
            }
        } catch (...) {
            poly_b200_sharded_destroy(h.release());
            throw;
        }
        h->m = pq->m;
        h->dim = (uint32_t)pq->dim;
        h->cb = pq->m;
        h->code_bits = pq->m * 8;
        *out = h.release();
    });
}

int poly_b200_sharded_destroy(poly_b200_sharded* h) {
    if (!h) return POLY_B200_OK;
    return guard([&] {
        free_staging(h);
        for (size_t g = 0; g < h->st.size(); ++g) {
            DeviceGuard dg(h->devices[g]);
            if (h->st[g].stream) cudaStreamDestroy(h->st[g].stream);
            if (h->st[g].done) cudaEventDestroy(h->st[g].done);
        }
        for (auto* ix : h->shards) poly_b200_destroy(ix);
        delete h;
    });
}

uint64_t poly_b200_sharded_size(const poly_b200_sharded* h) { return h ? h->n : 0; }
uint32_t poly_b200_sharded_count(const poly_b200_sharded* h) { return h ? (uint32_t)h->shards.size() : 0; }

int poly_b200_sharded_shard_size(const poly_b200_sharded* h, uint32_t shard, uint64_t* n) {
    return guard([&] {
        require(h && n && shard < h->shards.size(), POLY_B200_INVALID_ARGUMENT, "bad arguments");
        *n = poly_b200_size(h->shards[shard]);
    });
}

int poly_b200_sharded_add(poly_b200_sharded* h, const float* x, uint64_t n, const int64_t* ids) {
    return guard([&] {
        require(h != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        require(n == 0 || x, POLY_B200_INVALID_ARGUMENT, "null vectors");
        std::lock_guard<std::mutex> lk(h->mu);
        if (n == 0) return;
        for (uint64_t i = 0; i < n * h->dim; ++i)
            require(std::isfinite(x[i]), POLY_B200_INVALID_ARGUMENT, "non-finite entry in vector set");
        std::vector<int64_t> seq;
        if (!ids) {  // FlatIndex::add: ids default to size() + i
            seq.resize(n);
            for (uint64_t i = 0; i < n; ++i) seq[i] = (int64_t)(h->n + i);
            ids = seq.data();
        }
        const size_t P = h->shards.size();
        for_shards(h, [&](size_t g) {
            const uint64_t a = part_lo(n, P, g), b = part_lo(n, P, g + 1);
            rethrow(poly_b200_add(h->shards[g], x + a * h->dim, b - a, ids + a));
        });
        h->n += n;
    });
}

int poly_b200_sharded_add_codes(poly_b200_sharded* h, const uint8_t* codes, const int64_t* ids, uint64_t n) {
    return guard([&] {
        require(h != nullptr, POLY_B200_INVALID_ARGUMENT, "null index");
        require(n == 0 || codes, POLY_B200_INVALID_ARGUMENT, "null codes");
        std::lock_guard<std::mutex> lk(h->mu);
        if (n == 0) return;
        std::vector<int64_t> seq;
        if (!ids) {
            seq.resize(n);
            for (uint64_t i = 0; i < n; ++i) seq[i] = (int64_t)(h->n + i);
            ids = seq.data();
        }
        const size_t P = h->shards.size();
        for_shards(h, [&](size_t g) {
            const uint64_t a = part_lo(n, P, g), b = part_lo(n, P, g + 1);
            rethrow(poly_b200_add_codes(h->shards[g], codes + a * h->cb, ids + a, b - a));
        });
        h->n += n;
    });
}

int poly_b200_sharded_search_batch(poly_b200_sharded* h, const float* queries, uint64_t nq,
                                   const poly_b200_search_params* p, int64_t* out_ids, float* out_scores,
                                   uint32_t* out_counts, poly_b200_search_stats* stats) {
    return guard([&] {
        require(h != nullptr && p != nullptr, POLY_B200_INVALID_ARGUMENT, "null arguments");
        require(p->strategy >= 0 && p->strategy <= 3, POLY_B200_INVALID_ARGUMENT, "unknown strategy");
        require(p->tau <= h->code_bits, POLY_B200_INVALID_ARGUMENT, "tau exceeds code bits");
        require(p->k <= (uint32_t)pb::KMAX, POLY_B200_INVALID_ARGUMENT, "k > 2048 is not supported on the GPU path");
        require(nq == 0 || queries, POLY_B200_INVALID_ARGUMENT, "null queries");
        require(nq == 0 || p->k == 0 || (out_ids && out_scores), POLY_B200_INVALID_ARGUMENT, "null outputs");
        std::lock_guard<std::mutex> lk(h->mu);
        if (stats) *stats = {0, 0};
        if (nq == 0) return;
        const uint32_t k = p->k;
        if (k == 0) {  // SPEC: k = 0 returns empty lists
            if (out_counts) std::memset(out_counts, 0, nq * 4);
            if (stats) stats->scanned = h->n * nq;
            return;
        }
        const size_t P = h->shards.size();
        ensure_staging(h, nq, k);
        std::vector<poly_b200_search_stats> sst(P);
        // every shard: queries in, K1 / K2s / K2 / K3 on its device, its top-k stays there
        for_shards(h, [&](size_t g) {
            DeviceGuard dg(h->devices[g]);
            auto& s = h->st[g];
            CK(cudaMemcpyAsync(s.d_q, queries, nq * h->dim * 4, cudaMemcpyHostToDevice, s.stream));
            rethrow(poly_b200_search_batch_device(h->shards[g], s.d_q, nq, p, s.d_ids, s.d_sc, s.d_cnt, nullptr,
                                                  s.stream, stats ? &sst[g] : nullptr));
            CK(cudaEventRecord(s.done, s.stream));
        });
        // merge on devices[0].  K3g reads the shards' lists in place over peer memory when every
        // shard is loadable from devices[0] and a query's lists fit a warp's shared memory; otherwise
        // the lists are gathered with peer copies first and merged by K3m.
        DeviceGuard dg(h->devices[0]);
        cudaStream_t s0 = h->st[0].stream;
        for (size_t g = 0; g < P; ++g) CK(cudaStreamWaitEvent(s0, h->st[g].done, 0));
        const size_t gm_warp = ((P * (size_t)k * 12 + 15) & ~(size_t)15) + (size_t)pb::GM_PARTS * 4, gm_smem = gm_warp * pb::GM_WARPS;
        bool fused = P <= pb::GM_PARTS && gm_smem <= 200 * 1024;
        for (size_t g = 0; g < P; ++g) fused = fused && h->direct[g];
        if (fused) {
            pb::GatherSrc src{};
            for (size_t g = 0; g < P; ++g) {
                src.ids[g] = h->st[g].d_ids;
                src.sc[g] = h->st[g].d_sc;
                src.cnt[g] = h->st[g].d_cnt;
            }
            CK(cudaFuncSetAttribute(pb::gather_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gm_smem));
            pb::gather_merge_kernel<<<(unsigned)((nq + pb::GM_WARPS - 1) / pb::GM_WARPS), pb::GM_WARPS * 32, gm_smem, s0>>>(
                src, (uint32_t)P, (uint32_t)nq, k, h->o_ids, h->o_sc, h->o_cnt);
        } else {
            for (size_t g = 0; g < P; ++g) {
                auto& s = h->st[g];
                const size_t off = g * nq * k;
                CK(cudaMemcpyPeerAsync(h->g_ids + off, h->devices[0], s.d_ids, h->devices[g], nq * k * 8, s0));
                CK(cudaMemcpyPeerAsync(h->g_sc + off, h->devices[0], s.d_sc, h->devices[g], nq * k * 4, s0));
                CK(cudaMemcpyPeerAsync(h->g_cnt + g * nq, h->devices[0], s.d_cnt, h->devices[g], nq * 4, s0));
            }
            pb::merge_sorted_kernel<<<(unsigned)((nq + 127) / 128), 128, 0, s0>>>(
                h->g_ids, h->g_sc, h->g_cnt, (uint32_t)P, (uint32_t)nq, k, h->o_ids, h->o_sc, h->o_cnt);
        }
        pb::count_launch();
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out_ids, h->o_ids, nq * k * 8, cudaMemcpyDeviceToHost, s0));
        CK(cudaMemcpyAsync(out_scores, h->o_sc, nq * k * 4, cudaMemcpyDeviceToHost, s0));
        if (out_counts) CK(cudaMemcpyAsync(out_counts, h->o_cnt, nq * 4, cudaMemcpyDeviceToHost, s0));
        CK(cudaStreamSynchronize(s0));
        if (stats)
            for (auto& x : sst) {
                stats->scanned += x.scanned;
                stats->survivors += x.survivors;
            }
    });
}

}  // extern "C"
