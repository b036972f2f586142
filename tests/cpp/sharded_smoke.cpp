// C++ caller of the multi-GPU FlatIndex mirror (poly_b200::ShardedFlatIndex): the same
// inputs as mirror_smoke.cpp, rows spread over the shards of the given devices, ids
// global; prints the top-10 ids per query and the summed statistics.
#include <cstdio>
#include <cstdlib>
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
    if (argc < 5) return 2;
    const size_t n = 20000, nq = 24, dim = 128;
    poly_b200::ProductQuantizer pq;
    pq.m = 8;
    pq.dbits = 8;
    pq.dim = dim;
    pq.codebooks = slurp<float>(argv[1], 8 * 256 * 16);
    pq.perms = slurp<uint16_t>(argv[2], 8 * 256);
    auto blob = slurp<uint8_t>(argv[3], n * 8 + nq * dim * 4);
    std::vector<int> devices(std::atoi(argv[4]), 0);
    poly_b200::ShardedFlatIndex index(pq, devices);
    index.add_codes(blob.data(), nullptr, n / 2);  // two add calls: each one is split over the shards
    index.add_codes(blob.data() + (n / 2) * 8, nullptr, n - n / 2);
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
    return 0;
}
