// host_common.h -- host-side helpers shared by the flat (capi.cu) and IVF
// (capi_ivf.cu) C ABIs: poly::errc-style errors that never cross the C
// boundary as exceptions (common.hpp:13-40), device allocation, and the id map.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/poly_b200.h"
#include "poly_b200.cuh"

namespace pbh {

extern thread_local std::string g_err;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void require(bool ok, int code, const std::string& msg) {
    if (!ok) throw Error(code, msg);
}

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(POLY_B200_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ::pbh::ck((x), #x)

template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        return POLY_B200_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return POLY_B200_INTERNAL;
    }
}

template <class T>
T* dalloc(size_t count) {
    void* p = nullptr;
    if (count) CK(cudaMalloc(&p, count * sizeof(T)));
    return static_cast<T*>(p);
}

inline void dfree(void* p) {
    if (p) cudaFree(p);
}

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// ProductQuantizer::validate (pq.cpp:130-149) for the shapes the GPU path supports.
inline void check_pq(const poly_b200_pq_desc* pq) {
    require(pq && pq->codebooks && pq->perms, POLY_B200_INVALID_ARGUMENT, "null product quantizer");
    require(pq->dbits == 8, POLY_B200_INVALID_ARGUMENT, "only dbits = 8 is supported on the GPU path");
    require(pq->m == 8 || pq->m == 16, POLY_B200_INVALID_ARGUMENT, "m must be 8 or 16 (64- or 128-bit codes)");
    require(pq->dim == (uint64_t)pq->m * pb::DSUB, POLY_B200_INVALID_ARGUMENT,
            "dim must be 16 * m (sub-vectors of 16 dimensions)");
    const size_t ks = 256;
    for (uint32_t sq = 0; sq < pq->m; ++sq) {  // pq.cpp:11-27: perms must be bijections
        std::vector<bool> seen(ks, false);
        for (size_t j = 0; j < ks; ++j) {
            const uint16_t v = pq->perms[sq * ks + j];
            require(v < ks && !seen[v], POLY_B200_INVALID_ARGUMENT,
                    "assignment for sub-quantizer " + std::to_string(sq) + " is not a bijection");
            seen[v] = true;
        }
    }
    for (size_t i = 0; i < (size_t)pq->m * ks * pb::DSUB; ++i)
        require(std::isfinite(pq->codebooks[i]), POLY_B200_INVALID_ARGUMENT, "non-finite codebook entry");
}

// Ids of the stored vectors in insertion order (int64, Neighbor::id,
// flat_index.hpp:39-42) and their device form: the 32-bit key low word.
//   arithmetic ids (id0 + i, the default)  -> key low = id0 + i, no table
//   other ids in [0, 2^32)                  -> key low = id (uint32 table)
//   anything else                           -> key low = rank of the id, and a
//                                              rank -> id table maps back
// Keys order exactly like (score, id) in every mode.
struct IdMap {
    bool arith = true;
    int64_t id0 = 0;
    std::vector<int64_t> h;  // materialised ids once not arithmetic
    bool dirty = true;
    int mode = pb::ID_ARITH;
    uint32_t key_id0 = 0;
    uint32_t* d_id32 = nullptr;
    int64_t* d_rank_to_id = nullptr;

    void append(const int64_t* ids, uint64_t base, uint64_t n) {
        if (arith) {
            const int64_t first = (base == 0 && ids && n) ? ids[0] : id0;
            bool seq = true;
            if (ids)
                for (uint64_t i = 0; i < n && seq; ++i) seq = ids[i] == first + (int64_t)(base + i);
            if (seq) {
                id0 = first;
                dirty = true;
                return;
            }
            arith = false;
            h.resize(base);
            std::iota(h.begin(), h.end(), id0);
        }
        const size_t old = h.size();
        h.resize(old + n);
        for (uint64_t i = 0; i < n; ++i) h[old + i] = ids ? ids[i] : (int64_t)(base + i);
        dirty = true;
    }

    void append_range(int64_t first, uint64_t base, uint64_t n) {
        if (arith && (base == 0 || first == id0 + (int64_t)base)) {
            if (base == 0) id0 = first;
            dirty = true;
            return;
        }
        std::vector<int64_t> ids(n);
        std::iota(ids.begin(), ids.end(), first);
        append(ids.data(), base, n);
    }

    int64_t at(uint64_t i) const { return arith ? id0 + (int64_t)i : h[i]; }

    void release() {
        dfree(d_id32);
        dfree(d_rank_to_id);
        d_id32 = nullptr;
        d_rank_to_id = nullptr;
    }

    // Upload the device form for positions [0, n).
    void sync(uint64_t n) {
        if (!dirty) return;
        release();
        if (arith && id0 >= 0 && id0 + (int64_t)n <= (int64_t)UINT32_MAX + 1) {
            mode = pb::ID_ARITH;
            key_id0 = (uint32_t)id0;
        } else {
            std::vector<int64_t> tmp;
            if (arith) {
                tmp.resize(n);
                std::iota(tmp.begin(), tmp.end(), id0);
            }
            const std::vector<int64_t>& I = arith ? tmp : h;
            require(n <= (uint64_t)UINT32_MAX + 1, POLY_B200_INVALID_ARGUMENT, "more than 2^32 codes per device");
            std::vector<uint32_t> id32(n);
            const bool small =
                std::all_of(I.begin(), I.begin() + n, [](int64_t v) { return v >= 0 && v <= (int64_t)UINT32_MAX; });
            if (small) {
                for (uint64_t i = 0; i < n; ++i) id32[i] = (uint32_t)I[i];
            } else {
                std::vector<uint32_t> order(n);
                std::iota(order.begin(), order.end(), 0u);
                std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return I[a] < I[b]; });
                std::vector<int64_t> r2id(n);
                for (uint64_t r = 0; r < n; ++r) {
                    id32[order[r]] = (uint32_t)r;
                    r2id[r] = I[order[r]];
                }
                d_rank_to_id = dalloc<int64_t>(std::max<uint64_t>(n, 1));
                if (n) CK(cudaMemcpy(d_rank_to_id, r2id.data(), n * 8, cudaMemcpyHostToDevice));
            }
            d_id32 = dalloc<uint32_t>(std::max<uint64_t>(n, 1));
            if (n) CK(cudaMemcpy(d_id32, id32.data(), n * 4, cudaMemcpyHostToDevice));
            mode = pb::ID_TABLE;
        }
        dirty = false;
    }
};

}  // namespace pbh
