// poly_b200/flat_index.hpp -- C++ mirror of poly::FlatIndex over the C ABI.
//
// Same names, argument meaning and error behaviour as the reference class
// (/root/reference/proj/include/poly/flat_index.hpp:39-144, errors
// common.hpp:13-40): a reference caller switches by changing the namespace
// and linking libpoly_b200.so.  ProductQuantizer here carries only the fields
// the search path consumes (pq.hpp:49-60).
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../poly_b200.h"

namespace poly_b200 {

enum class errc { ok = 0, invalid_argument, io, format, state, corrupt, version, internal };  // common.hpp:13-22

class error : public std::runtime_error {  // common.hpp:25-32
public:
    error(errc code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
    errc code() const noexcept { return code_; }

private:
    errc code_;
};

inline void check(int rc) {
    if (rc != POLY_B200_OK) throw error(static_cast<errc>(rc), poly_b200_last_error());
}

struct Neighbor {  // flat_index.hpp:39-42
    std::int64_t id;
    float score;
};

enum class Strategy { adc = POLY_B200_ADC, binary = POLY_B200_BINARY, disidx = POLY_B200_DISIDX, dual = POLY_B200_DUAL };

inline Strategy strategy_from_string(const std::string& name) {
    if (name == "adc") return Strategy::adc;
    if (name == "binary") return Strategy::binary;
    if (name == "disidx") return Strategy::disidx;
    if (name == "dual") return Strategy::dual;
    throw error(errc::invalid_argument, "unknown strategy '" + name + "'");
}

inline const char* to_string(Strategy s) {
    switch (s) {
        case Strategy::adc: return "adc";
        case Strategy::binary: return "binary";
        case Strategy::disidx: return "disidx";
        default: return "dual";
    }
}

struct SearchParams {  // flat_index.hpp:48-52
    Strategy strategy = Strategy::adc;
    std::uint32_t k = 10;
    std::uint32_t tau = 0;
};

struct SearchStats {  // flat_index.hpp:54-57
    std::uint64_t scanned = 0;
    std::uint64_t survivors = 0;
};

struct ProductQuantizer {  // pq.hpp:49-60 (fields used by the search path)
    std::uint32_t m = 0;
    std::uint32_t dbits = 0;
    std::size_t dim = 0;
    std::vector<float> codebooks;        // m * ksub * dsub
    std::vector<std::uint16_t> perms;    // m * ksub: centroid index -> stored field
    std::uint32_t ksub() const { return 1u << dbits; }
    std::size_t dsub() const { return dim / m; }
    std::size_t code_bits() const { return static_cast<std::size_t>(m) * dbits; }
    std::size_t code_bytes() const { return (code_bits() + 7) / 8; }
};

struct VectorSet {  // vectors.hpp:12-32 (row-major data + ids)
    std::vector<float> data;
    std::vector<std::int64_t> ids;
    std::size_t dim = 0;
    std::size_t size() const { return dim == 0 ? 0 : data.size() / dim; }
};

class FlatIndex {  // flat_index.hpp:99-144
public:
    FlatIndex() = default;
    explicit FlatIndex(ProductQuantizer pq, int device = 0) : pq_(std::move(pq)) {
        poly_b200_pq_desc d{pq_.m, pq_.dbits, pq_.dim, pq_.codebooks.data(), pq_.perms.data()};
        check(poly_b200_create(&d, device, &h_));
    }
    FlatIndex(const FlatIndex&) = delete;
    FlatIndex& operator=(const FlatIndex&) = delete;
    FlatIndex(FlatIndex&& o) noexcept : pq_(std::move(o.pq_)), default_tau(o.default_tau), h_(o.h_) { o.h_ = nullptr; }
    FlatIndex& operator=(FlatIndex&& o) noexcept {
        if (this != &o) {
            poly_b200_destroy(h_);
            pq_ = std::move(o.pq_);
            default_tau = o.default_tau;
            h_ = o.h_;
            o.h_ = nullptr;
        }
        return *this;
    }
    ~FlatIndex() { poly_b200_destroy(h_); }

    const ProductQuantizer& pq() const { return pq_; }
    std::size_t size() const { return poly_b200_size(h_); }
    std::size_t code_bytes() const { return pq_.code_bytes(); }
    std::uint32_t code_bits() const { return static_cast<std::uint32_t>(pq_.code_bits()); }

    std::vector<std::uint8_t> codes() const {
        std::vector<std::uint8_t> out(size() * code_bytes());
        check(poly_b200_get_codes(h_, out.data(), nullptr));
        return out;
    }
    std::vector<std::int64_t> ids() const {
        std::vector<std::int64_t> out(size());
        check(poly_b200_get_codes(h_, nullptr, out.data()));
        return out;
    }

    std::optional<std::uint32_t> default_tau;  // flat_index.hpp:113

    /// Encodes (on the GPU) and appends; ids come from the set.
    void add(const VectorSet& x, unsigned /*threads*/ = 0) {
        if (x.dim != pq_.dim) throw error(errc::invalid_argument, "encode dimension mismatch");
        check(poly_b200_add(h_, x.data.data(), x.size(), x.ids.empty() ? nullptr : x.ids.data()));
    }

    /// Appends pre-encoded codes (serialization path).
    void add_codes(const std::uint8_t* codes, const std::int64_t* ids, std::size_t n) {
        check(poly_b200_add_codes(h_, codes, ids, n));
    }

    std::vector<Neighbor> search(const float* query, const SearchParams& params, SearchStats* stats = nullptr) const {
        return std::move(run(query, 1, params, stats)[0]);
    }

    std::vector<std::vector<Neighbor>> search_batch(const VectorSet& queries, const SearchParams& params,
                                                    unsigned /*threads*/ = 0,
                                                    SearchStats* total_stats = nullptr) const {
        if (queries.dim != pq_.dim) throw error(errc::invalid_argument, "query dimension mismatch");
        return run(queries.data.data(), queries.size(), params, total_stats);
    }

    std::uint32_t calibrate_threshold(const VectorSet& train_queries, double target_filter_rate,
                                      bool* warning = nullptr, unsigned /*threads*/ = 0) const {
        std::uint32_t tau = 0;
        int w = 0;
        check(poly_b200_calibrate_threshold(h_, train_queries.data.data(), train_queries.size(), target_filter_rate,
                                            &tau, &w));
        if (warning) *warning = w != 0;
        return tau;
    }

    FlatIndex with_assignments(const std::vector<std::uint16_t>& perms) const {
        FlatIndex out;
        out.pq_ = pq_;
        out.pq_.perms = perms;
        check(poly_b200_with_assignments(h_, perms.data(), &out.h_));
        return out;
    }

    poly_b200_index* handle() const { return h_; }

private:
    std::vector<std::vector<Neighbor>> run(const float* q, std::size_t nq, const SearchParams& p,
                                           SearchStats* stats) const {
        const poly_b200_search_params cp{static_cast<std::int32_t>(p.strategy), p.k, p.tau};
        std::vector<std::int64_t> ids(nq * p.k);
        std::vector<float> scores(nq * p.k);
        std::vector<std::uint32_t> counts(nq);
        poly_b200_search_stats st{0, 0};
        check(poly_b200_search_batch(h_, q, nq, &cp, ids.data(), scores.data(), counts.data(), &st));
        if (stats) {
            stats->scanned += st.scanned;
            stats->survivors += st.survivors;
        }
        std::vector<std::vector<Neighbor>> out(nq);
        for (std::size_t i = 0; i < nq; ++i) {
            out[i].resize(counts[i]);
            for (std::uint32_t r = 0; r < counts[i]; ++r) out[i][r] = {ids[i * p.k + r], scores[i * p.k + r]};
        }
        return out;
    }

    ProductQuantizer pq_;
    poly_b200_index* h_ = nullptr;
};

/// FlatIndex over several GPUs of this process (poly_b200_sharded_*): one shard per
/// entry of `devices`; add / add_codes split their rows across the shards, search
/// merges the per-shard top-k on devices[0].  Same results as FlatIndex over the union.
class ShardedFlatIndex {
public:
    ShardedFlatIndex(ProductQuantizer pq, const std::vector<int>& devices) : pq_(std::move(pq)) {
        poly_b200_pq_desc d{pq_.m, pq_.dbits, pq_.dim, pq_.codebooks.data(), pq_.perms.data()};
        check(poly_b200_sharded_create(&d, devices.data(), static_cast<std::uint32_t>(devices.size()), &h_));
    }
    ShardedFlatIndex(const ShardedFlatIndex&) = delete;
    ShardedFlatIndex& operator=(const ShardedFlatIndex&) = delete;
    ~ShardedFlatIndex() { poly_b200_sharded_destroy(h_); }

    const ProductQuantizer& pq() const { return pq_; }
    std::size_t size() const { return poly_b200_sharded_size(h_); }
    std::size_t shards() const { return poly_b200_sharded_count(h_); }

    void add(const VectorSet& x, unsigned /*threads*/ = 0) {
        if (x.dim != pq_.dim) throw error(errc::invalid_argument, "encode dimension mismatch");
        check(poly_b200_sharded_add(h_, x.data.data(), x.size(), x.ids.empty() ? nullptr : x.ids.data()));
    }
    void add_codes(const std::uint8_t* codes, const std::int64_t* ids, std::size_t n) {
        check(poly_b200_sharded_add_codes(h_, codes, ids, n));
    }

    std::vector<Neighbor> search(const float* query, const SearchParams& params, SearchStats* stats = nullptr) const {
        return std::move(run(query, 1, params, stats)[0]);
    }
    std::vector<std::vector<Neighbor>> search_batch(const VectorSet& queries, const SearchParams& params,
                                                    unsigned /*threads*/ = 0,
                                                    SearchStats* total_stats = nullptr) const {
        if (queries.dim != pq_.dim) throw error(errc::invalid_argument, "query dimension mismatch");
        return run(queries.data.data(), queries.size(), params, total_stats);
    }

private:
    std::vector<std::vector<Neighbor>> run(const float* q, std::size_t nq, const SearchParams& p,
                                           SearchStats* stats) const {
        const poly_b200_search_params cp{static_cast<std::int32_t>(p.strategy), p.k, p.tau};
        std::vector<std::int64_t> ids(nq * p.k);
        std::vector<float> scores(nq * p.k);
        std::vector<std::uint32_t> counts(nq);
        poly_b200_search_stats st{0, 0};
        check(poly_b200_sharded_search_batch(h_, q, nq, &cp, ids.data(), scores.data(), counts.data(), &st));
        if (stats) {
            stats->scanned += st.scanned;
            stats->survivors += st.survivors;
        }
        std::vector<std::vector<Neighbor>> out(nq);
        for (std::size_t i = 0; i < nq; ++i) {
            out[i].resize(counts[i]);
            for (std::uint32_t r = 0; r < counts[i]; ++r) out[i][r] = {ids[i * p.k + r], scores[i * p.k + r]};
        }
        return out;
    }

    ProductQuantizer pq_;
    poly_b200_sharded* h_ = nullptr;
};

}  // namespace poly_b200
