// Exercises the C++ mirror of poly::FlatIndex (include/poly_b200/flat_index.hpp)
// the way a reference caller would: reads a PQ, codes and queries written by the
// test, runs search_batch / search / calibrate_threshold and prints the results.
#include <cstdio>
#include <fstream>
#include <vector>

#include "poly_b200/flat_index.hpp"

template <class T>
static std::vector<T> slurp(const char* path, size_t n) {
    std::vector<T> v(n);
    std::ifstream f(path, std::ios::binary);
    f.read(reinterpret_cast<char*>(v.data()), n * sizeof(T));
    return v;
}

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    const size_t n = 20000, nq = 24, dim = 128;
    poly_b200::ProductQuantizer pq;
    pq.m = 8;
    pq.dbits = 8;
    pq.dim = dim;
    pq.codebooks = slurp<float>(argv[1], 8 * 256 * 16);
    pq.perms = slurp<uint16_t>(argv[2], 8 * 256);
    auto blob = slurp<uint8_t>(argv[3], n * 8 + nq * dim * 4);
    poly_b200::FlatIndex index(pq, 0);
    index.add_codes(blob.data(), nullptr, n);
    poly_b200::VectorSet q;
    q.dim = dim;
    q.data.assign(reinterpret_cast<const float*>(blob.data() + n * 8),
                  reinterpret_cast<const float*>(blob.data() + n * 8) + nq * dim);
    poly_b200::SearchParams p{poly_b200::Strategy::dual, 10, 24};
    poly_b200::SearchStats st;
    auto res = index.search_batch(q, p, 0, &st);
    std::printf("stats %llu %llu\n", (unsigned long long)st.scanned, (unsigned long long)st.survivors);
    for (auto& r : res) {
        for (auto& nb : r) std::printf("%lld ", (long long)nb.id);
        std::printf("\n");
    }
    try {
        poly_b200::SearchParams bad{poly_b200::Strategy::dual, 10, 65};
        index.search(q.data.data(), bad);
        std::printf("no error\n");
    } catch (const poly_b200::error& e) {
        std::printf("error %d\n", (int)e.code());
    }
    std::printf("tau95 %u\n", index.calibrate_threshold(q, 0.95));
    return 0;
}
