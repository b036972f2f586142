/* polyoracle.c -- CPU restatement of the polysemous search path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline.  The product path
 * (paper_1609_01882_b200/, libpoly_b200.so) never links or calls it.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks every function below
 * against golden vectors produced by the reference's own compiled sources
 * (oracle/_ref/libpolyref.so, built by oracle/Makefile from
 * /root/reference/proj/src; fixtures in tests/golden/ with the generating
 * script tests/golden/make_golden.py).
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj unless they start with SPEC.md).  Compile with
 * -ffp-contract=off: the reference sums are plain fp32 adds/muls in a fixed
 * order (objdump of the reference build shows vsubss/vmulss/vaddss, no FMA). */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PO_OK 0
#define PO_EINVAL 1

/* ------------------------------------------------------------------------- */
/* Synthetic Gaussian-mixture generator (not a reference function).           */
/* Counter-based so that any row can be produced independently; the GPU       */
/* generator in paper_1609_01882_b200/csrc/synth.cuh computes the identical  */
/* bits (integer hashing, an exact int->float conversion and IEEE adds/muls). */
/* N(0,1) is approximated by Irwin-Hall(12): sum of 12 uniforms minus 6.      */
/* ------------------------------------------------------------------------- */
static inline uint64_t po_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t po_hash64(uint64_t x) { return po_mix64(x); }

static inline uint64_t po_row_key(uint64_t seed, uint32_t stream, uint64_t row) {
    const uint64_t base = po_mix64(seed + 0x632BE59BD9B4E019ull * (uint64_t)(stream + 1));
    return po_mix64(base ^ (row * 0xD1B54A32D192ED03ull));
}

static inline float po_normal(uint64_t rowkey, uint32_t t) {
    uint64_t s = 0;
    for (uint32_t j = 0; j < 6; ++j) {
        const uint64_t h = po_mix64(rowkey ^ ((uint64_t)(6u * t + j + 1u) * 0xA0761D6478BD642Full));
        s += (h >> 40) + ((h >> 16) & 0xFFFFFFull);
    }
    const int64_t c = (int64_t)s - (int64_t)6 * 16777216;
    return (float)c * (1.0f / 16777216.0f);
}

/* Mixture centers: C[c][t] = 10 * N(0,1), stream 0. */
void po_gen_centers(uint64_t seed, uint32_t ncent, uint32_t dim, float* out) {
    for (uint32_t c = 0; c < ncent; ++c) {
        const uint64_t key = po_row_key(seed, 0, c);
        for (uint32_t t = 0; t < dim; ++t) out[(size_t)c * dim + t] = 10.0f * po_normal(key, t);
    }
}

/* Rows [row0, row0+n) of stream `stream` (1 train, 2 base, 3 queries):
 * x = max(0, C[u] + N(0,1)), u uniform over centers; optional unit norm. */
void po_gen_points(uint64_t seed, uint32_t stream, uint64_t row0, uint64_t n, const float* centers,
                   uint32_t ncent, uint32_t dim, int normalize, float* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t key = po_row_key(seed, stream, row0 + i);
        const uint32_t u = (uint32_t)(((po_mix64(key ^ 0x5851F42D4C957F2Dull) >> 32) * (uint64_t)ncent) >> 32);
        float* x = out + i * dim;
        float nrm = 0.0f;
        for (uint32_t t = 0; t < dim; ++t) {
            const float v = centers[(size_t)u * dim + t] + po_normal(key, t);
            x[t] = v > 0.0f ? v : 0.0f;
            nrm += x[t] * x[t];
        }
        if (normalize) {
            const float inv = nrm > 0.0f ? 1.0f / sqrtf(nrm) : 0.0f;
            for (uint32_t t = 0; t < dim; ++t) x[t] = x[t] * inv;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* PQ primitives                                                              */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint32_t m, dbits, dim;
    const float* codebooks;   /* m * ksub * dsub   (pq.hpp:53) */
    const uint16_t* perms;    /* m * ksub: centroid -> field (pq.hpp:54) */
    const uint16_t* inv_perms;/* m * ksub: field -> centroid (pq.hpp:55) */
} po_pq;

static inline uint32_t po_ksub(const po_pq* pq) { return 1u << pq->dbits; }
static inline uint32_t po_dsub(const po_pq* pq) { return pq->dim / pq->m; }
static inline uint32_t po_code_bits(const po_pq* pq) { return pq->m * pq->dbits; }
static inline uint32_t po_code_bytes(const po_pq* pq) { return (po_code_bits(pq) + 7) / 8; }

/* pq.hpp:24-31 */
static inline uint32_t po_get_field(const uint8_t* code, uint32_t m, uint32_t dbits) {
    const size_t bit = (size_t)m * dbits;
    const size_t byte = bit >> 3;
    const unsigned shift = (unsigned)(bit & 7);
    uint32_t w = code[byte];
    if (shift + dbits > 8) w |= (uint32_t)code[byte + 1] << 8;
    return (w >> shift) & ((1u << dbits) - 1u);
}

/* pq.hpp:33-43 */
static inline void po_set_field(uint8_t* code, uint32_t m, uint32_t dbits, uint32_t value) {
    const size_t bit = (size_t)m * dbits;
    const size_t byte = bit >> 3;
    const unsigned shift = (unsigned)(bit & 7);
    const uint32_t mask = (1u << dbits) - 1u;
    uint32_t w = code[byte];
    if (shift + dbits > 8) w |= (uint32_t)code[byte + 1] << 8;
    w = (w & ~(mask << shift)) | ((value & mask) << shift);
    code[byte] = (uint8_t)(w & 0xff);
    if (shift + dbits > 8) code[byte + 1] = (uint8_t)((w >> 8) & 0xff);
}

/* distances.cpp:10-17 */
float po_sq_l2(const float* a, const float* b, size_t dim) {
    float acc = 0.0f;
    for (size_t i = 0; i < dim; ++i) {
        const float d = a[i] - b[i];
        acc += d * d;
    }
    return acc;
}

/* pq.cpp:91-105: lut[sq][j] = sq_l2(q_sq, c_{sq,j}), indexed by centroid j. */
void po_compute_lut(const po_pq* pq, const float* q, float* lut) {
    const uint32_t ks = po_ksub(pq), ds = po_dsub(pq);
    for (uint32_t sq = 0; sq < pq->m; ++sq)
        for (uint32_t j = 0; j < ks; ++j)
            lut[(size_t)sq * ks + j] = po_sq_l2(q + (size_t)sq * ds, pq->codebooks + ((size_t)sq * ks + j) * ds, ds);
}

/* pq.cpp:107-119: lutp[sq][f] = lut[sq][inv_perm[sq][f]], indexed by stored field. */
void po_permuted_lut(const po_pq* pq, const float* lut, float* lutp) {
    const uint32_t ks = po_ksub(pq);
    for (uint32_t sq = 0; sq < pq->m; ++sq)
        for (uint32_t f = 0; f < ks; ++f)
            lutp[(size_t)sq * ks + f] = lut[(size_t)sq * ks + pq->inv_perms[(size_t)sq * ks + f]];
}

/* pq.cpp:29-45: argmin with strict <, ties keep the lowest index; store perm[best]. */
void po_encode(const po_pq* pq, const float* x, uint8_t* code) {
    const uint32_t ks = po_ksub(pq), ds = po_dsub(pq);
    memset(code, 0, po_code_bytes(pq));
    for (uint32_t sq = 0; sq < pq->m; ++sq) {
        const float* sub = x + (size_t)sq * ds;
        const float* cb = pq->codebooks + (size_t)sq * ks * ds;
        uint32_t best = 0;
        float best_d = po_sq_l2(sub, cb, ds);
        for (uint32_t j = 1; j < ks; ++j) {
            const float d = po_sq_l2(sub, cb + (size_t)j * ds, ds);
            if (d < best_d) { best_d = d; best = j; }
        }
        po_set_field(code, sq, pq->dbits, pq->perms[(size_t)sq * ks + best]);
    }
}

/* flat_index.hpp:14-27 */
uint32_t po_hamming_bytes(const uint8_t* a, const uint8_t* b, size_t nbytes) {
    uint32_t acc = 0;
    size_t i = 0;
    for (; i + 8 <= nbytes; i += 8) {
        uint64_t wa, wb;
        memcpy(&wa, a + i, 8);
        memcpy(&wb, b + i, 8);
        acc += (uint32_t)__builtin_popcountll(wa ^ wb);
    }
    for (; i < nbytes; ++i) acc += (uint32_t)__builtin_popcount((unsigned)(a[i] ^ b[i]));
    return acc;
}

/* flat_index.hpp:30-37 */
uint32_t po_disidx(const uint8_t* a, const uint8_t* b, uint32_t m, uint32_t dbits) {
    uint32_t acc = 0;
    for (uint32_t sq = 0; sq < m; ++sq) acc += po_get_field(a, sq, dbits) != po_get_field(b, sq, dbits);
    return acc;
}

/* pq.cpp:121-128: acc = 0; acc += lut[sq][inv_perm[sq][field_sq]] in sq order. */
float po_adc_distance(const po_pq* pq, const float* lut, const uint8_t* code) {
    const uint32_t ks = po_ksub(pq);
    float acc = 0.0f;
    for (uint32_t sq = 0; sq < pq->m; ++sq) {
        const uint32_t f = po_get_field(code, sq, pq->dbits);
        acc += lut[(size_t)sq * ks + pq->inv_perms[(size_t)sq * ks + f]];
    }
    return acc;
}

/* Same sum through the permuted table (pq.hpp:83 "for direct scans"); bit-identical
 * to po_adc_distance because the terms and their order are the same. */
static inline float po_adc_permuted(const po_pq* pq, const float* lutp, const uint8_t* code) {
    const uint32_t ks = po_ksub(pq);
    float acc = 0.0f;
    for (uint32_t sq = 0; sq < pq->m; ++sq) acc += lutp[(size_t)sq * ks + po_get_field(code, sq, pq->dbits)];
    return acc;
}

/* ------------------------------------------------------------------------- */
/* Top-k per the SPEC contract: the k lexicographically */
/* smallest (score, id), ascending.  NOT the reference TopK class               */
/* (flat_index.hpp:60-94), whose heap comparator is inverted. */
/* A bounded max-heap whose root is the worst kept element.                    */
/* ------------------------------------------------------------------------- */
typedef struct { float score; int64_t id; } po_nb;

static inline int po_worse(po_nb a, po_nb b) {  /* flat_index.hpp:88-90 */
    return a.score > b.score || (a.score == b.score && a.id > b.id);
}

static void po_sift_down(po_nb* h, size_t n, size_t i) {
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, w = i;
        if (l < n && po_worse(h[l], h[w])) w = l;
        if (r < n && po_worse(h[r], h[w])) w = r;
        if (w == i) return;
        po_nb t = h[i]; h[i] = h[w]; h[w] = t;
        i = w;
    }
}

static void po_sift_up(po_nb* h, size_t i) {
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (!po_worse(h[i], h[p])) return;
        po_nb t = h[i]; h[i] = h[p]; h[p] = t;
        i = p;
    }
}

typedef struct { po_nb* h; size_t n, k; } po_topk;

static inline void po_topk_offer(po_topk* t, float score, int64_t id) {
    if (t->k == 0) return;
    po_nb x = {score, id};
    if (t->n < t->k) { t->h[t->n] = x; po_sift_up(t->h, t->n); t->n++; return; }
    if (po_worse(t->h[0], x)) { t->h[0] = x; po_sift_down(t->h, t->n, 0); }
}

static int po_cmp_nb(const void* a, const void* b) {
    const po_nb* x = (const po_nb*)a; const po_nb* y = (const po_nb*)b;
    if (po_worse(*y, *x)) return -1;
    if (po_worse(*x, *y)) return 1;
    return 0;
}

/* Brute-force check helper exposed for the top-k unit test. */
uint32_t po_topk_select(const float* scores, const int64_t* ids, uint64_t n, uint32_t k, int64_t* out_ids,
                        float* out_scores) {
    po_topk t = {(po_nb*)malloc(sizeof(po_nb) * (k ? k : 1)), 0, k};
    for (uint64_t i = 0; i < n; ++i) po_topk_offer(&t, scores[i], ids[i]);
    qsort(t.h, t.n, sizeof(po_nb), po_cmp_nb);
    for (size_t i = 0; i < t.n; ++i) { out_ids[i] = t.h[i].id; out_scores[i] = t.h[i].score; }
    uint32_t n_out = (uint32_t)t.n;
    free(t.h);
    return n_out;
}

/* ------------------------------------------------------------------------- */
/* parallel_chunks restated (common.cpp:8-39): contiguous chunks of [0,n) on   */
/* min(threads, n) threads, chunk boundaries depend only on (n, threads).      */
/* ------------------------------------------------------------------------- */
typedef void (*po_chunk_fn)(void* ctx, size_t begin, size_t end);
typedef struct { po_chunk_fn fn; void* ctx; size_t b, e; } po_job;
static void* po_job_run(void* p) { po_job* j = (po_job*)p; j->fn(j->ctx, j->b, j->e); return NULL; }

static void po_parallel_chunks(size_t n, unsigned threads, po_chunk_fn fn, void* ctx) {
    if (n == 0) return;
    if (threads == 0) threads = 1;
    size_t nch = threads < n ? threads : n;
    if (nch == 1) { fn(ctx, 0, n); return; }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nch);
    po_job* jobs = (po_job*)malloc(sizeof(po_job) * nch);
    size_t base = n / nch, extra = n % nch, b = 0;
    for (size_t c = 0; c < nch; ++c) {
        size_t len = base + (c < extra ? 1 : 0);
        jobs[c].fn = fn; jobs[c].ctx = ctx; jobs[c].b = b; jobs[c].e = b + len;
        pthread_create(&th[c], NULL, po_job_run, &jobs[c]);
        b += len;
    }
    for (size_t c = 0; c < nch; ++c) pthread_join(th[c], NULL);
    free(th); free(jobs);
}

/* ------------------------------------------------------------------------- */
/* Search (FlatIndex::search / search_batch, flat_index.hpp:121-126; declared  */
/* but not defined in the reference).  Restated from SPEC.md:303-317 (operation),*/
/* :335-339 (two full passes, shortage -> survivors only, ties -> lower id,    */
/* parallel over queries) and :328-333 (invariants).                           */
/* strategy: 0 adc, 1 binary, 2 disidx, 3 dual (flat_index.hpp:44).            */
/* ------------------------------------------------------------------------- */
typedef struct {
    const po_pq* pq; const uint8_t* codes; const int64_t* ids; uint64_t n;
    const float* queries; int strategy; uint32_t k, tau;
    int64_t* out_ids; float* out_scores; uint32_t* out_counts;
    uint64_t* out_survivors; uint64_t* out_survivor_hash;
} po_search_ctx;

static void po_search_chunk(void* p, size_t qb, size_t qe) {
    po_search_ctx* c = (po_search_ctx*)p;
    const po_pq* pq = c->pq;
    const uint32_t ks = po_ksub(pq), cb = po_code_bytes(pq);
    float* lut = (float*)malloc(sizeof(float) * pq->m * ks);
    float* lutp = (float*)malloc(sizeof(float) * pq->m * ks);
    uint8_t* qcode = (uint8_t*)malloc(cb);
    uint32_t* surv = (uint32_t*)malloc(sizeof(uint32_t) * (c->n ? c->n : 1));
    po_topk t = {(po_nb*)malloc(sizeof(po_nb) * (c->k ? c->k : 1)), 0, c->k};
    for (size_t qi = qb; qi < qe; ++qi) {
        const float* q = c->queries + qi * pq->dim;
        t.n = 0;
        uint64_t nsurv = 0, hsurv = 0;
        if (c->k > 0 && c->n > 0) {
            po_encode(pq, q, qcode);            /* pq.cpp:29-45 */
            po_compute_lut(pq, q, lut);         /* pq.cpp:91-105 */
            po_permuted_lut(pq, lut, lutp);     /* pq.cpp:107-119 */
            if (c->strategy == 3) {
                /* pass 1: survivors = {i : hamming <= tau} */
                for (uint64_t i = 0; i < c->n; ++i)
                    if (po_hamming_bytes(qcode, c->codes + i * cb, cb) <= c->tau) surv[nsurv++] = (uint32_t)i;
                /* pass 2: ADC rerank of survivors, top-k by (score, id) */
                for (uint64_t s = 0; s < nsurv; ++s) {
                    const uint64_t i = surv[s];
                    hsurv += po_mix64((uint64_t)c->ids[i]);  /* survivor-set hash: sum of mix64(id) */
                    po_topk_offer(&t, po_adc_permuted(pq, lutp, c->codes + i * cb), c->ids[i]);
                }
            } else {
                for (uint64_t i = 0; i < c->n; ++i) {
                    const uint8_t* code = c->codes + i * cb;
                    float s;
                    if (c->strategy == 0) s = po_adc_permuted(pq, lutp, code);
                    else if (c->strategy == 1) s = (float)po_hamming_bytes(qcode, code, cb);
                    else s = (float)po_disidx(qcode, code, pq->m, pq->dbits);
                    po_topk_offer(&t, s, c->ids[i]);
                }
            }
        }
        qsort(t.h, t.n, sizeof(po_nb), po_cmp_nb);
        for (uint32_t r = 0; r < c->k; ++r) {
            c->out_ids[qi * c->k + r] = r < t.n ? t.h[r].id : -1;
            c->out_scores[qi * c->k + r] = r < t.n ? t.h[r].score : INFINITY;
        }
        c->out_counts[qi] = (uint32_t)t.n;
        if (c->out_survivors) c->out_survivors[qi] = nsurv;
        if (c->out_survivor_hash) c->out_survivor_hash[qi] = hsurv;
    }
    free(lut); free(lutp); free(qcode); free(surv); free(t.h);
}

int po_search_batch(uint32_t m, uint32_t dbits, uint32_t dim, const float* codebooks, const uint16_t* perms,
                    const uint16_t* inv_perms, const uint8_t* codes, const int64_t* ids, uint64_t n,
                    const float* queries, uint64_t nq, int strategy, uint32_t k, uint32_t tau, unsigned threads,
                    int64_t* out_ids, float* out_scores, uint32_t* out_counts, uint64_t* out_survivors,
                    uint64_t* out_survivor_hash) {
    po_pq pq = {m, dbits, dim, codebooks, perms, inv_perms};
    if (m == 0 || dbits < 1 || dbits > 8 || dim % m != 0 || strategy < 0 || strategy > 3) return PO_EINVAL;
    if (tau > m * dbits) return PO_EINVAL;
    po_search_ctx c = {&pq, codes, ids, n, queries, strategy, k, tau, out_ids, out_scores, out_counts,
                       out_survivors, out_survivor_hash};
    po_parallel_chunks(nq, threads, po_search_chunk, &c);
    return PO_OK;
}

/* ------------------------------------------------------------------------- */
/* Batch helpers used by the parity tests                                     */
/* ------------------------------------------------------------------------- */
typedef struct { const po_pq* pq; const float* x; uint8_t* codes; } po_enc_ctx;
static void po_encode_chunk(void* p, size_t b, size_t e) {
    po_enc_ctx* c = (po_enc_ctx*)p;
    const uint32_t cb = po_code_bytes(c->pq);
    for (size_t i = b; i < e; ++i) po_encode(c->pq, c->x + i * c->pq->dim, c->codes + i * cb);
}

/* FlatIndex::add (flat_index.hpp:115-116) restated as per-vector encode
 * (pq.cpp:29-45).  The reference's encode_batch (pq.cpp:47-78) goes through
 * a BLAS GEMM and can flip near-ties; the product encoder matches encode(). */
void po_encode_batch(uint32_t m, uint32_t dbits, uint32_t dim, const float* codebooks, const uint16_t* perms,
                     const float* x, uint64_t n, uint8_t* codes, unsigned threads) {
    po_pq pq = {m, dbits, dim, codebooks, perms, NULL};
    po_enc_ctx c = {&pq, x, codes};
    po_parallel_chunks(n, threads, po_encode_chunk, &c);
}

/* LUT (centroid-indexed), permuted LUT and query code for a batch of queries. */
void po_lut_batch(uint32_t m, uint32_t dbits, uint32_t dim, const float* codebooks, const uint16_t* perms,
                  const uint16_t* inv_perms, const float* q, uint64_t nq, float* lut, float* lutp, uint8_t* qcodes) {
    po_pq pq = {m, dbits, dim, codebooks, perms, inv_perms};
    const size_t L = (size_t)m << dbits;
    for (uint64_t i = 0; i < nq; ++i) {
        po_compute_lut(&pq, q + i * dim, lut + i * L);
        if (lutp) po_permuted_lut(&pq, lut + i * L, lutp + i * L);
        if (qcodes) po_encode(&pq, q + i * dim, qcodes + i * po_code_bytes(&pq));
    }
}

/* Hamming histogram per query: hist[q][h] = #codes at distance h (0..code_bits). */
typedef struct { const po_pq* pq; const uint8_t* codes; uint64_t n; const float* q; uint64_t* hist; } po_hist_ctx;
static void po_hist_chunk(void* p, size_t b, size_t e) {
    po_hist_ctx* c = (po_hist_ctx*)p;
    const uint32_t cb = po_code_bytes(c->pq), nb = po_code_bits(c->pq) + 1;
    uint8_t* qc = (uint8_t*)malloc(cb);
    for (size_t i = b; i < e; ++i) {
        po_encode(c->pq, c->q + i * c->pq->dim, qc);
        uint64_t* h = c->hist + i * nb;
        memset(h, 0, sizeof(uint64_t) * nb);
        for (uint64_t j = 0; j < c->n; ++j) h[po_hamming_bytes(qc, c->codes + j * cb, cb)]++;
    }
    free(qc);
}

void po_hamming_histogram(uint32_t m, uint32_t dbits, uint32_t dim, const float* codebooks, const uint16_t* perms,
                          const uint8_t* codes, uint64_t n, const float* q, uint64_t nq, unsigned threads,
                          uint64_t* hist) {
    po_pq pq = {m, dbits, dim, codebooks, perms, NULL};
    po_hist_ctx c = {&pq, codes, n, q, hist};
    po_parallel_chunks(nq, threads, po_hist_chunk, &c);
}

/* FlatIndex::calibrate_threshold (flat_index.hpp:128-132):
 * max { tau : mean survivor fraction over train queries <= 1 - rate };
 * returns 0 with *warning = 1 when even tau = 0 keeps too many. */
uint32_t po_calibrate_from_histogram(const uint64_t* hist, uint64_t nq, uint32_t code_bits, uint64_t n,
                                     double rate, int* warning) {
    if (warning) *warning = 0;
    const uint32_t nb = code_bits + 1;
    double cum = 0.0;
    int64_t best = -1;
    for (uint32_t tau = 0; tau < nb; ++tau) {
        for (uint64_t i = 0; i < nq; ++i) cum += (double)hist[i * nb + tau];
        const double frac = (nq && n) ? cum / ((double)nq * (double)n) : 0.0;
        if (frac <= 1.0 - rate) best = tau;
    }
    if (best < 0) { if (warning) *warning = 1; return 0; }
    return (uint32_t)best;
}

/* FlatIndex::with_assignments (flat_index.hpp:134-136): relabel each field
 * f -> new_perm[old_inv_perm[f]], exactly as if re-encoded. */
void po_relabel_codes(uint32_t m, uint32_t dbits, const uint16_t* old_inv_perms, const uint16_t* new_perms,
                      uint8_t* codes, uint64_t n) {
    const uint32_t ks = 1u << dbits, cb = (m * dbits + 7) / 8;
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t sq = 0; sq < m; ++sq) {
            const uint32_t f = po_get_field(codes + i * cb, sq, dbits);
            po_set_field(codes + i * cb, sq, dbits, new_perms[(size_t)sq * ks + old_inv_perms[(size_t)sq * ks + f]]);
        }
}

/* ------------------------------------------------------------------------- */
/* IVF (coarseindex; no reference code exists).              */
/* Restated from reference primitives: sq_l2 (distances.cpp:10-17), encode   */
/* (pq.cpp:29-45), compute_lut/permuted_lut (pq.cpp:91-119), hamming_bytes    */
/* (flat_index.hpp:14-27) and the SPEC top-k contract.                        */
/*   build: every vector goes to its nearest coarse cell    */
/*     (sq_l2, strict <, ties -> lowest cell); residual r = x - c (fp32).     */
/*   enumerate_cells: the nprobe cells with the smallest    */
/*     sq_l2(q, c), ascending; ties -> lower cell id.                         */
/*   search_coarse: visit cells in that order; per cell the */
/*     query residual q - c gets its own code and LUT; dual */
/*     filter + ADC over the cell's (id, residual code) list; stop after the  */
/*     cell at which the scanned count reaches cap (cap counts pre-filter     */
/*     codes; 0 = no cap); global top-k over visited cells.      */
/* ------------------------------------------------------------------------- */
typedef struct { const float* x; uint32_t dim; const float* cent; uint32_t nlist; uint32_t* assign; } po_asg_ctx;
static void po_assign_chunk(void* p, size_t b, size_t e) {
    po_asg_ctx* c = (po_asg_ctx*)p;
    for (size_t i = b; i < e; ++i) {
        const float* xi = c->x + i * c->dim;
        uint32_t best = 0;
        float bd = po_sq_l2(xi, c->cent, c->dim);
        for (uint32_t j = 1; j < c->nlist; ++j) {
            const float d = po_sq_l2(xi, c->cent + (size_t)j * c->dim, c->dim);
            if (d < bd) { bd = d; best = j; }
        }
        c->assign[i] = best;
    }
}

void po_ivf_assign(const float* x, uint64_t n, uint32_t dim, const float* centroids, uint32_t nlist, unsigned threads,
                   uint32_t* assign) {
    po_asg_ctx c = {x, dim, centroids, nlist, assign};
    po_parallel_chunks(n, threads, po_assign_chunk, &c);
}

typedef struct { float d; uint32_t c; } po_cd;
static int po_cmp_cd(const void* a, const void* b) {
    const po_cd* x = (const po_cd*)a; const po_cd* y = (const po_cd*)b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return x->c < y->c ? -1 : (x->c > y->c);
}

typedef struct {
    const po_pq* pq; const float* cent; uint32_t nlist; const uint64_t* off; const uint8_t* codes; const int64_t* ids;
    const float* queries; uint32_t nprobe; uint64_t cap; int strategy; uint32_t k, tau;
    int64_t* out_ids; float* out_scores; uint32_t* out_counts; uint64_t* out_surv; uint64_t* out_scanned;
    uint32_t* out_probes; uint64_t* out_surv_hash;
} po_ivf_ctx;

static void po_ivf_chunk(void* p, size_t qb, size_t qe) {
    po_ivf_ctx* c = (po_ivf_ctx*)p;
    const po_pq* pq = c->pq;
    const uint32_t ks = po_ksub(pq), cb = po_code_bytes(pq), dim = pq->dim;
    po_cd* cd = (po_cd*)malloc(sizeof(po_cd) * c->nlist);
    float* r = (float*)malloc(sizeof(float) * dim);
    float* lut = (float*)malloc(sizeof(float) * pq->m * ks);
    float* lutp = (float*)malloc(sizeof(float) * pq->m * ks);
    uint8_t* qcode = (uint8_t*)malloc(cb);
    po_topk t = {(po_nb*)malloc(sizeof(po_nb) * (c->k ? c->k : 1)), 0, c->k};
    for (size_t qi = qb; qi < qe; ++qi) {
        const float* q = c->queries + qi * dim;
        t.n = 0;
        uint64_t nsurv = 0, nscan = 0, hsurv = 0;
        uint32_t visited = 0;
        if (c->k > 0) {
            for (uint32_t j = 0; j < c->nlist; ++j) { cd[j].d = po_sq_l2(q, c->cent + (size_t)j * dim, dim); cd[j].c = j; }
            qsort(cd, c->nlist, sizeof(po_cd), po_cmp_cd);
            const uint32_t np = c->nprobe < c->nlist ? c->nprobe : c->nlist;
            for (uint32_t pi = 0; pi < np; ++pi) {
                if (c->cap && nscan >= c->cap) break;
                const uint32_t cell = cd[pi].c;
                const float* cc = c->cent + (size_t)cell * dim;
                for (uint32_t d = 0; d < dim; ++d) r[d] = q[d] - cc[d];
                po_encode(pq, r, qcode);
                po_compute_lut(pq, r, lut);
                po_permuted_lut(pq, lut, lutp);
                for (uint64_t i = c->off[cell]; i < c->off[cell + 1]; ++i) {
                    const uint8_t* code = c->codes + i * cb;
                    float s;
                    if (c->strategy == 3) {
                        if (po_hamming_bytes(qcode, code, cb) > c->tau) continue;
                        ++nsurv;
                        hsurv += po_mix64((uint64_t)c->ids[i]);
                        s = po_adc_permuted(pq, lutp, code);
                    } else if (c->strategy == 0) s = po_adc_permuted(pq, lutp, code);
                    else if (c->strategy == 1) s = (float)po_hamming_bytes(qcode, code, cb);
                    else s = (float)po_disidx(qcode, code, pq->m, pq->dbits);
                    po_topk_offer(&t, s, c->ids[i]);
                }
                nscan += c->off[cell + 1] - c->off[cell];
                ++visited;
            }
        }
        qsort(t.h, t.n, sizeof(po_nb), po_cmp_nb);
        for (uint32_t rr = 0; rr < c->k; ++rr) {
            c->out_ids[qi * c->k + rr] = rr < t.n ? t.h[rr].id : -1;
            c->out_scores[qi * c->k + rr] = rr < t.n ? t.h[rr].score : INFINITY;
        }
        c->out_counts[qi] = (uint32_t)t.n;
        if (c->out_surv) c->out_surv[qi] = nsurv;
        if (c->out_surv_hash) c->out_surv_hash[qi] = hsurv;
        if (c->out_scanned) c->out_scanned[qi] = nscan;
        if (c->out_probes) {
            const uint32_t np = c->nprobe < c->nlist ? c->nprobe : c->nlist;
            for (uint32_t pi = 0; pi < c->nprobe; ++pi) c->out_probes[qi * c->nprobe + pi] = pi < np ? cd[pi].c : 0xFFFFFFFFu;
        }
    }
    free(cd); free(r); free(lut); free(lutp); free(qcode); free(t.h);
}

int po_ivf_search(uint32_t m, uint32_t dbits, uint32_t dim, const float* codebooks, const uint16_t* perms,
                  const uint16_t* inv_perms, const float* centroids, uint32_t nlist, const uint64_t* list_off,
                  const uint8_t* list_codes, const int64_t* list_ids, const float* queries, uint64_t nq, uint32_t nprobe,
                  uint64_t cap, int strategy, uint32_t k, uint32_t tau, unsigned threads, int64_t* out_ids,
                  float* out_scores, uint32_t* out_counts, uint64_t* out_survivors, uint64_t* out_scanned,
                  uint32_t* out_probes, uint64_t* out_survivor_hash) {
    po_pq pq = {m, dbits, dim, codebooks, perms, inv_perms};
    if (m == 0 || dbits < 1 || dbits > 8 || dim % m != 0 || strategy < 0 || strategy > 3 || nlist == 0) return PO_EINVAL;
    if (tau > m * dbits || nprobe == 0) return PO_EINVAL;
    po_ivf_ctx c = {&pq, centroids, nlist, list_off, list_codes, list_ids, queries, nprobe, cap, strategy, k, tau,
                    out_ids, out_scores, out_counts, out_survivors, out_scanned, out_probes, out_survivor_hash};
    po_parallel_chunks(nq, threads, po_ivf_chunk, &c);
    return PO_OK;
}

/* Residual codes of the build: encode(x - c_assign). */
void po_ivf_encode_residuals(uint32_t m, uint32_t dbits, uint32_t dim, const float* codebooks, const uint16_t* perms,
                             const float* x, uint64_t n, const float* centroids, const uint32_t* assign, uint8_t* codes) {
    po_pq pq = {m, dbits, dim, codebooks, perms, NULL};
    float* r = (float*)malloc(sizeof(float) * dim);
    for (uint64_t i = 0; i < n; ++i) {
        const float* cc = centroids + (size_t)assign[i] * dim;
        for (uint32_t d = 0; d < dim; ++d) r[d] = x[i * dim + d] - cc[d];
        po_encode(&pq, r, codes + i * po_code_bytes(&pq));
    }
    free(r);
}
