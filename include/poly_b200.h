/* poly_b200.h -- C ABI of the B200 polysemous-code search path.
 *
 * Drop-in boundary for the reference's flat index
 * (/root/reference/proj/include/poly/flat_index.hpp:99-144, class poly::FlatIndex).
 * Plain pointers and sizes only; no exceptions cross this boundary.  Every
 * entry point returns a status from the reference's error space
 * (common.hpp:13-22, "usable across the C boundary" common.hpp:24) and leaves a
 * message in poly_b200_last_error().  A C++ mirror of poly::FlatIndex built on
 * these calls is in include/poly_b200/flat_index.hpp; the Python mirror is
 * paper_1609_01882_b200.FlatIndex.
 *
 * Scope: dbits = 8 (one byte per sub-quantizer field, the layout of
 * every configuration), m in {8, 16} (64- and 128-bit codes), k <= 2048.
 * Other shapes are rejected with POLY_B200_INVALID_ARGUMENT.
 */
#ifndef POLY_B200_H
#define POLY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* poly::errc (common.hpp:13-22) */
enum poly_b200_status {
    POLY_B200_OK = 0,
    POLY_B200_INVALID_ARGUMENT = 1,
    POLY_B200_IO = 2,
    POLY_B200_FORMAT = 3,
    POLY_B200_STATE = 4,
    POLY_B200_CORRUPT = 5,
    POLY_B200_VERSION = 6,
    POLY_B200_INTERNAL = 7
};

/* poly::Strategy (flat_index.hpp:44) */
enum poly_b200_strategy { POLY_B200_ADC = 0, POLY_B200_BINARY = 1, POLY_B200_DISIDX = 2, POLY_B200_DUAL = 3 };

/* poly::ProductQuantizer (pq.hpp:49-89): codebooks m x 2^dbits x dim/m fp32,
 * perms m x 2^dbits (centroid index -> stored field). */
typedef struct {
    uint32_t m;
    uint32_t dbits;
    uint64_t dim;
    const float* codebooks;
    const uint16_t* perms;
} poly_b200_pq_desc;

/* poly::SearchParams (flat_index.hpp:48-52) */
typedef struct {
    int32_t strategy;
    uint32_t k;
    uint32_t tau;
} poly_b200_search_params;

/* poly::SearchStats (flat_index.hpp:54-57) */
typedef struct {
    uint64_t scanned;
    uint64_t survivors;
} poly_b200_search_stats;

typedef struct poly_b200_index poly_b200_index;

/* Message of the last failing call on this thread ("" if none). */
const char* poly_b200_last_error(void);

/* FlatIndex(ProductQuantizer) (flat_index.hpp:102).  `device` is the CUDA
 * ordinal; the PQ tables are copied to it. */
int poly_b200_create(const poly_b200_pq_desc* pq, int device, poly_b200_index** out);
int poly_b200_destroy(poly_b200_index* index);

/* size() / code_bytes() / code_bits() (flat_index.hpp:105-107) */
uint64_t poly_b200_size(const poly_b200_index* index);
uint32_t poly_b200_code_bytes(const poly_b200_index* index);

/* FlatIndex::add (flat_index.hpp:115-116): encode n host vectors (n x dim fp32)
 * on the GPU and append.  ids may be NULL (sequential from size()). */
int poly_b200_add(poly_b200_index* index, const float* x, uint64_t n, const int64_t* ids);

/* FlatIndex::add_codes (flat_index.hpp:118-119): append n pre-encoded host codes
 * (n x code_bytes) with their ids (NULL = sequential from size()). */
int poly_b200_add_codes(poly_b200_index* index, const uint8_t* codes, const int64_t* ids, uint64_t n);

/* FlatIndex::search_batch (flat_index.hpp:124-126), host buffers.
 * queries nq x dim fp32; out_ids / out_scores nq x k (unfilled slots: id -1,
 * score +inf); out_counts nq (may be NULL); stats summed over queries (may be NULL).
 * FlatIndex::search (flat_index.hpp:121-122) is the nq = 1 case. */
int poly_b200_search_batch(poly_b200_index* index, const float* queries, uint64_t nq,
                           const poly_b200_search_params* params, int64_t* out_ids, float* out_scores,
                           uint32_t* out_counts, poly_b200_search_stats* stats);

/* Same, with every buffer in device memory of the index's device and work
 * enqueued on `stream` (a cudaStream_t, NULL = legacy default stream).
 * Per-query survivor counts go to out_survivors (device, nq, may be NULL).
 * Returns after enqueueing; `stats` (host, may be NULL) forces a sync. */
int poly_b200_search_batch_device(poly_b200_index* index, const float* d_queries, uint64_t nq,
                                  const poly_b200_search_params* params, int64_t* d_out_ids, float* d_out_scores,
                                  uint32_t* d_out_counts, uint64_t* d_out_survivors, void* stream,
                                  poly_b200_search_stats* stats);

/* Same, plus the per-query survivor-set hash: out_survivor_hash[q] = sum over the
 * codes that pass the dual filter of mix64(id) mod 2^64 (splitmix64 finaliser,
 * order-independent; the parity suite compares it with the oracle's).  Either
 * per-query output may be NULL; strategies other than dual report 0. */
int poly_b200_search_batch_device_ex(poly_b200_index* index, const float* d_queries, uint64_t nq,
                                     const poly_b200_search_params* params, int64_t* d_out_ids, float* d_out_scores,
                                     uint32_t* d_out_counts, uint64_t* d_out_survivors,
                                     uint64_t* d_out_survivor_hash, void* stream, poly_b200_search_stats* stats);

/* FlatIndex::calibrate_threshold (flat_index.hpp:128-132):
 * max { tau : mean survivor fraction over the train queries <= 1 - rate };
 * returns 0 in *tau with *warning = 1 when even tau = 0 keeps too many. */
int poly_b200_calibrate_threshold(poly_b200_index* index, const float* train_queries, uint64_t nq,
                                  double target_filter_rate, uint32_t* tau, int* warning);

/* FlatIndex::with_assignments (flat_index.hpp:134-136): new index over the same
 * codebooks and vectors under new perms (m x 2^dbits); codes are relabeled
 * field by field exactly as if re-encoded. */
int poly_b200_with_assignments(const poly_b200_index* index, const uint16_t* perms, poly_b200_index** out);

/* Copy the stored codes (n x code_bytes) / ids back to host (FlatIndex::codes(), ids()). */
int poly_b200_get_codes(const poly_b200_index* index, uint8_t* codes, int64_t* ids);

/* ---- multi-GPU plumbing ----------------------------
 * Per-shard search that stops before mapping keys to ids: writes, per query,
 * up to k 64-bit keys (fp32 score bits << 32 | 32-bit id rank) ascending, and
 * the key count.  All ranks all-gather these and call poly_b200_merge_keys. */
int poly_b200_search_keys_device(poly_b200_index* index, const float* d_queries, uint64_t nq,
                                 const poly_b200_search_params* params, uint64_t* d_out_keys, uint32_t* d_out_counts,
                                 uint64_t* d_out_survivors, void* stream);

/* Merge `parts` key lists per query (layout parts x nq x k, counts parts x nq)
 * into the global top-k; keys are mapped to ids by the index's id map
 * (the shards of one logical index share it). */
int poly_b200_merge_keys_device(poly_b200_index* index, const uint64_t* d_keys, const uint32_t* d_counts,
                                uint32_t parts, uint64_t nq, uint32_t k, int64_t* d_out_ids, float* d_out_scores,
                                uint32_t* d_out_counts, void* stream);

/* Synthetic workload generator used by the benchmark and the large-N tests:
 * appends rows [row0, row0 + n) of the seeded Gaussian mixture (stream_id),
 * generated and encoded on the GPU (never materialised); bit-identical to
 * oracle/polyoracle.c po_gen_points followed by encode (pq.cpp:29-45).
 * The appended ids are the global row numbers row0 .. row0 + n - 1, so the
 * shards of one database keep globally consistent ids. */
int poly_b200_add_synthetic(poly_b200_index* index, uint64_t seed, const float* centers, uint32_t ncent,
                            uint32_t stream_id, uint64_t row0, uint64_t n, int normalize);

/* Device-side generator of float rows (same stream definition), for tests. */
int poly_b200_gen_points_device(int device, uint64_t seed, const float* centers, uint32_t ncent, uint32_t dim,
                                uint32_t stream_id, uint64_t row0, uint64_t n, int normalize, float* d_out,
                                void* stream);

/* Test hook: K1 only -- stored-field LUTs (nq x m x 256 fp32, permuted_lut
 * pq.cpp:107-119) and query codes (nq x code_bytes, encode pq.cpp:29-45) for
 * host queries, copied back to host buffers. */
int poly_b200_debug_lut(poly_b200_index* index, const float* queries, uint64_t nq, float* lutp, uint8_t* qcodes);

/* Test hook: per-query candidate counts and final thresholds of the last
 * scanned batch (nq <= 256 entries each). */
int poly_b200_debug_counts(poly_b200_index* index, uint32_t* ccount, uint64_t* thr, uint32_t nq);

/* Test hooks for the candidate-list overflow path: force the per-query candidate
 * list capacity (rounded to the select block; 0 = default), and count the queries
 * of the last batch whose list overflowed and were re-ranked by the exact rescue
 * scan (kernels_rescue.cu).  IVF twins below. */
int poly_b200_debug_set_list_capacity(poly_b200_index* index, uint32_t cap);
int poly_b200_debug_rescued(poly_b200_index* index, uint32_t* n_rescued);

/* Timing hook for bench.py: while enabled, CUDA events bracket every K2 scan
 * launch on its stream; poly_b200_profile_read waits for them and returns the
 * summed K2 time (ms) and launch count since the last read. */
int poly_b200_profile_enable(poly_b200_index* index, int enable);
int poly_b200_profile_read(poly_b200_index* index, double* scan_ms, uint64_t* scan_launches);

/* ---- IVF + polysemous (coarseindex; configs 2 and 4) ------
 * Coarse quantizer of nlist centroids (nlist x dim fp32); inverted lists of
 * (id, residual code) where the residual PQ (`pq`) encodes x - c_cell.
 * enumerate_cells: the nprobe cells with the smallest sq_l2(q, c), ascending,
 * ties -> lower cell.  search_coarse: per probed cell the query residual gets
 * its own code and LUT; dual filter + ADC over the list; cells are visited in
 * order and the visit stops after the cell at which `cap` scanned codes is
 * reached (0 = no cap); global top-k.  The reference ships no IVF code; the
 * oracle restates SPEC from the reference's primitives. */
typedef struct poly_b200_ivf poly_b200_ivf;

typedef struct {
    int32_t strategy;
    uint32_t k;
    uint32_t tau;
    uint32_t nprobe;
    uint64_t cap;
} poly_b200_ivf_params;

int poly_b200_ivf_create(const poly_b200_pq_desc* pq, const float* coarse, uint32_t nlist, int device,
                         poly_b200_ivf** out);
int poly_b200_ivf_destroy(poly_b200_ivf* ivf);
uint64_t poly_b200_ivf_size(const poly_b200_ivf* ivf);

/* build: nearest cell by sq_l2 (strict <, lowest cell on
 * ties) for n host vectors -> cells (n). */
int poly_b200_ivf_assign(poly_b200_ivf* ivf, const float* x, uint64_t n, uint32_t* cells);

/* Assign, residual-encode and append n host vectors; ids may be NULL
 * (sequential from size()).  cells may be NULL (computed) or given. */
int poly_b200_ivf_add(poly_b200_ivf* ivf, const float* x, uint64_t n, const uint32_t* cells, const int64_t* ids);

/* Same for device-resident vectors and cells (cells required), ids
 * id0 .. id0 + n - 1; used by the benchmark's chunked builder. */
int poly_b200_ivf_add_device(poly_b200_ivf* ivf, const float* d_x, const uint32_t* d_cells, uint64_t n, int64_t id0,
                             void* stream);
/* Same with explicit host ids (n int64), e.g. a by-list shard's scattered rows. */
int poly_b200_ivf_add_device_ids(poly_b200_ivf* ivf, const float* d_x, const uint32_t* d_cells, uint64_t n,
                                 const int64_t* ids, void* stream);

/* Append pre-encoded residual codes with their cells and ids (serialization). */
int poly_b200_ivf_add_codes(poly_b200_ivf* ivf, const uint32_t* cells, const uint8_t* codes, const int64_t* ids,
                            uint64_t n);

/* Lists in CSR form: off (nlist + 1), codes (size x code_bytes), ids (size);
 * any output may be NULL. */
int poly_b200_ivf_get_lists(poly_b200_ivf* ivf, uint64_t* off, uint8_t* codes, int64_t* ids);

/* Inverted-list file: save writes the PQ tables, coarse
 * centroids, CSR offsets, residual codes and int64 ids as checksummed sections; load
 * creates an index on `device` from such a file.  Errors: POLY_B200_IO (open/write),
 * POLY_B200_FORMAT (magic, section layout, shape), POLY_B200_VERSION, POLY_B200_CORRUPT
 * (checksum, truncation, offsets) -- the poly::errc classes (common.hpp:13-22). */
int poly_b200_ivf_save(poly_b200_ivf* ivf, const char* path);
int poly_b200_ivf_load(const char* path, int device, poly_b200_ivf** out);

/* enumerate_cells for host queries: cells (nq x nprobe). */
int poly_b200_ivf_probes(poly_b200_ivf* ivf, const float* queries, uint64_t nq, uint32_t nprobe, uint32_t* cells);

/* search_coarse, host buffers (ids/scores nq x k; unfilled: -1 / +inf). */
int poly_b200_ivf_search(poly_b200_ivf* ivf, const float* queries, uint64_t nq, const poly_b200_ivf_params* params,
                         int64_t* out_ids, float* out_scores, uint32_t* out_counts, poly_b200_search_stats* stats);

/* Device buffers, work enqueued on `stream`; `stats` (host, may be NULL) syncs. */
int poly_b200_ivf_search_device(poly_b200_ivf* ivf, const float* d_queries, uint64_t nq,
                                const poly_b200_ivf_params* params, int64_t* d_out_ids, float* d_out_scores,
                                uint32_t* d_out_counts, void* stream, poly_b200_search_stats* stats);

/* Same with per-query survivor counts and survivor-set hashes (device, nq each,
 * either may be NULL; as poly_b200_search_batch_device_ex). */
int poly_b200_ivf_search_device_ex(poly_b200_ivf* ivf, const float* d_queries, uint64_t nq,
                                   const poly_b200_ivf_params* params, int64_t* d_out_ids, float* d_out_scores,
                                   uint32_t* d_out_counts, uint64_t* d_out_survivors, uint64_t* d_out_survivor_hash,
                                   void* stream, poly_b200_search_stats* stats);

/* Multi-GPU IVF: each rank holds every cell's lists for its id
 * range (shard by id within every list) and returns its per-query top-k as
 * 64-bit keys (fp32 score bits << 32 | 32-bit global id); the ranks' keys are
 * all-gathered and merged exactly by poly_b200_ivf_merge_keys_device.  Requires
 * consecutive ids below 2^32 (POLY_B200_STATE otherwise).  Layouts as
 * poly_b200_search_keys_device / poly_b200_merge_keys_device. */
int poly_b200_ivf_search_keys_device(poly_b200_ivf* ivf, const float* d_queries, uint64_t nq,
                                     const poly_b200_ivf_params* params, uint64_t* d_keys, uint32_t* d_counts,
                                     void* stream, poly_b200_search_stats* stats);
int poly_b200_ivf_merge_keys_device(poly_b200_ivf* ivf, const uint64_t* d_keys, const uint32_t* d_counts,
                                    uint32_t parts, uint64_t nq, uint32_t k, int64_t* d_ids, float* d_scores,
                                    uint32_t* d_out_counts, void* stream);
/* The coarse quantization split by query over the ranks (the replicated part of the
 * sharding above): a rank computes the probes of its query slice with
 * poly_b200_ivf_probe_keys_device -- nq x min(nprobe, nlist) keys (dist bits << 32 |
 * cell), ascending per query, exactly enumerate_cells -- the ranks
 * all-gather them, and each rank scans its shard with the given probes through
 * poly_b200_ivf_search_keys_probes_device (same outputs as
 * poly_b200_ivf_search_keys_device; d_probe_keys holds nq x min(params->nprobe, nlist)
 * keys). */
int poly_b200_ivf_probe_keys_device(poly_b200_ivf* ivf, const float* d_queries, uint64_t nq, uint32_t nprobe,
                                    uint64_t* d_probe_keys, void* stream);
int poly_b200_ivf_search_keys_probes_device(poly_b200_ivf* ivf, const float* d_queries, uint64_t nq,
                                            const poly_b200_ivf_params* params, const uint64_t* d_probe_keys,
                                            uint64_t* d_keys, uint32_t* d_counts, void* stream,
                                            poly_b200_search_stats* stats);

/* Two-phase shard search for by-list sharding, one batch (nq <= the
 * batch size), probes given (all-gathered):
 *   phase 1: round 1 over each query's FIRST probe only -- empty on every rank but the one
 *            owning that cell -- writes the local bound (k-th key + 1; all ones = none)
 *            to d_thr (nq uint64);
 *   (caller: d_thr <- min over the ranks; any rank's k-th key bounds the global k-th)
 *   phase 2: round 2 over the other probes under min(local bound, d_thr), then this
 *            shard's top-k keys as poly_b200_ivf_search_keys_probes_device writes them.
 * The merged result equals the unsharded search (the bound only prunes keys that cannot
 * be in the global top-k). */
int poly_b200_ivf_search_keys_phase_device(poly_b200_ivf* ivf, const float* d_queries, uint64_t nq,
                                           const poly_b200_ivf_params* params, const uint64_t* d_probe_keys, int phase,
                                           uint64_t* d_thr, uint64_t* d_keys, uint32_t* d_counts, void* stream,
                                           poly_b200_search_stats* stats);

/* The lists of selected cells only, CSR in the order of `cells`: off (ncells + 1),
 * codes (off[ncells] x code_bytes), ids; codes / ids may be NULL. */
int poly_b200_ivf_get_cells(poly_b200_ivf* ivf, const uint32_t* cells, uint32_t ncells, uint64_t* off, uint8_t* codes,
                            int64_t* ids);

/* Timing hook for bench.py (as poly_b200_profile_*): CUDA events around every K6
 * list-scan launch while enabled; read returns the summed ms and the launch count. */
int poly_b200_ivf_profile_enable(poly_b200_ivf* ivf, int enable);
int poly_b200_ivf_profile_read(poly_b200_ivf* ivf, double* scan_ms, uint64_t* scan_launches);

/* Queries per internal batch (default 2048).  A larger batch groups more (query, probe)
 * pairs on each inverted list, so the cell-major list scan reads a list once for more
 * queries (codes reused across the group), at the cost of scratch memory that grows
 * with the batch (probe keys, residual LUTs, candidate lists).  Setting it waits for
 * outstanding searches and frees the batch-sized scratch; no reference equivalent
 * (search_coarse SPEC.md:382-390 takes one query at a time). */
int poly_b200_ivf_set_batch(poly_b200_ivf* ivf, uint32_t queries_per_batch);
uint32_t poly_b200_ivf_batch(const poly_b200_ivf* ivf);

int poly_b200_ivf_debug_set_list_capacity(poly_b200_ivf* ivf, uint32_t cap);
int poly_b200_ivf_debug_rescued(poly_b200_ivf* ivf, uint32_t* n_rescued);

/* knn_graph: the k nearest neighbours of n vectors that are
 * themselves in the index (vector i has id id0 + i), self-match removed:
 * search_coarse with k + 1, then the row's own id is dropped (or, if absent,
 * the (k+1)-th result).  Device buffers: d_x n x dim, outputs n x k. */
int poly_b200_ivf_knn_graph_device(poly_b200_ivf* ivf, const float* d_x, uint64_t n, int64_t id0,
                                   const poly_b200_ivf_params* params, int64_t* d_out_ids, float* d_out_scores,
                                   uint32_t* d_out_counts, void* stream);

/* ---- one FlatIndex over several GPUs of one process (SURVEY.md sec. 8(b) create(pq, n_gpus))
 * The drop-in for a FlatIndex whose database is sharded across the GPUs of a node,
 * driven by one host process (no torch.distributed): `devices` lists the CUDA
 * ordinals, one shard each (an ordinal may repeat: several shards on one GPU).
 * add / add_codes (flat_index.hpp:115-119) split every call's rows into n_devices
 * contiguous parts, part g to shard g, each row keeping its global id (NULL ids =
 * size() + i).  search_batch (flat_index.hpp:124-126) runs every shard concurrently
 * on its own device and merges the per-shard top-k lists on devices[0] in (score, id)
 * order, reading them in place over peer memory (one gather + merge kernel; peer copies
 * first when a device cannot load from a peer): the result equals the single-index
 * search over the union of the shards.  Statistics are summed over the shards. */
typedef struct poly_b200_sharded poly_b200_sharded;
int poly_b200_sharded_create(const poly_b200_pq_desc* pq, const int* devices, uint32_t n_devices,
                             poly_b200_sharded** out);
int poly_b200_sharded_destroy(poly_b200_sharded* index);
uint64_t poly_b200_sharded_size(const poly_b200_sharded* index);
uint32_t poly_b200_sharded_count(const poly_b200_sharded* index);
int poly_b200_sharded_shard_size(const poly_b200_sharded* index, uint32_t shard, uint64_t* n);
int poly_b200_sharded_add(poly_b200_sharded* index, const float* x, uint64_t n, const int64_t* ids);
int poly_b200_sharded_add_codes(poly_b200_sharded* index, const uint8_t* codes, const int64_t* ids, uint64_t n);
int poly_b200_sharded_search_batch(poly_b200_sharded* index, const float* queries, uint64_t nq,
                                   const poly_b200_search_params* params, int64_t* out_ids, float* out_scores,
                                   uint32_t* out_counts, poly_b200_search_stats* stats);

/* train_coarse's k-means on the GPU (the reference kmeans is
 * proj/src/kmeans.cpp:14-137 with KmeansParams kmeans.hpp:10-14): k-means++ seeding with
 * the reference's Rng (mt19937_64) draws, `iters` Lloyd iterations (exact nearest-cell
 * assignment by fp32 sq_l2, ties to the lower cell; centroids = float(double sum / count);
 * empty cells take the farthest member of the largest cell), then a final assignment.
 * x: n x dim host floats; centroids: k x dim out; assign (n, may be NULL);
 * iteration_mse (iters, may be NULL): the objective before each update; mse: the final one.
 * n <= k: every point is a centroid, cells replicate points cyclically. */
int poly_b200_kmeans(const float* x, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed, int device,
                     float* centroids, uint32_t* assign, double* iteration_mse, double* mse);

/* ---- k-NN graph output sink ("streamed to the output sink", External
 * Interfaces: one record per vector -- id, neighbor count, then (neighbor id, score)
 * pairs -- in a sectioned binary file, plus an optional ivecs export of neighbor ids).
 * File: magic "POLYKNNG", u32 version 1, u32 k, u64 records, one section
 * { "RECORDS_", u64 bytes, u64 fnv1a64(payload), payload }, payload = records
 * { i64 id, u32 count, count x { i64 neighbor id, f32 score } } packed, little-endian.
 * ivecs: per record an int32 k, then k int32 neighbor ids (-1 pads).
 * write_device appends the graph rows of n stored vectors (device d_x, ids id0 ..):
 * knn_graph on the GPU step by step, each step's rows written while the next is
 * searched.  close patches the record count and checksum. */
typedef struct poly_b200_knn_writer poly_b200_knn_writer;
int poly_b200_knn_writer_open(const char* path, const char* ivecs_path, uint32_t k, poly_b200_knn_writer** out);
int poly_b200_ivf_knn_graph_write_device(poly_b200_ivf* ivf, poly_b200_knn_writer* writer, const float* d_x,
                                         uint64_t n, int64_t id0, const poly_b200_ivf_params* params, void* stream);
int poly_b200_knn_writer_close(poly_b200_knn_writer* writer, uint64_t* records);

/* Number of kernel launches this library has issued so far (for bench.py). */
uint64_t poly_b200_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* POLY_B200_H */
