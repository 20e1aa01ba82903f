/*
 * pqk_b200.h — C-ABI of the B200-native PQk-means compressed-domain Lloyd iteration.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `pqclust` (arXiv 1709.03708, /root/reference/pkg/src/pqclust).  The reference
 * is pure Python; its only plugin interface for this path is the assignment
 * strategy registry
 *
 *     AssignStrategy = Callable[[codes, centers, DistanceTables, threads], uint32 labels]
 *       (clustering.py:200, register_assignment_strategy clustering.py:207-216)
 *
 * and the functions with no hook that must be replaced by same-signature
 * functions: `fit` (clustering.py:377-482), `assign` (clustering.py:255-282),
 * `paired_distance_sq` (pq.py:271-290) and `encode` (pq.py:205-231).
 * Every entry point below takes plain pointers and sizes (no torch types) and
 * returns a pqk_status_t; the Python host layer maps PQK_EINVAL to ValueError and
 * everything else to RuntimeError, mirroring the reference error behaviour.
 *
 * Two levels:
 *   1. Host-buffer entry points (pqk_*_host): the calls a ctypes/cffi binding of
 *      the reference's strategy plugin makes.  Inputs and outputs are host memory
 *      (pageable or pinned); the library manages device buffers and one stream per
 *      device internally.  Synchronous on return.
 *   2. Device-pointer entry points (pqk_*_device): stream-ordered kernel launches on
 *      caller-owned device memory.  Used by the resident Lloyd engine (fit) and the
 *      multi-GPU driver, which allreduces the histogram between
 *      pqk_histogram_device and pqk_vote_device.
 *
 * Device code layout: codes and centers are row-major uint8 with a padded row
 * stride MP = pqk_padded_m(M) (pad bytes are 0; pad subspaces use all-zero
 * tables).  Tables are the reference's float64 (M, L, L) DistanceTables
 * (pq.py:64-95), C-contiguous.
 */
#ifndef PQK_B200_H
#define PQK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQK_ABI_VERSION 1

typedef enum {
  PQK_OK = 0,
  PQK_EINVAL = 1,       /* bad argument: maps to ValueError            */
  PQK_ECUDA = 2,        /* CUDA runtime / launch failure: RuntimeError */
  PQK_ENOMEM = 3,       /* device allocation failed: MemoryError       */
  PQK_EUNSUPPORTED = 4, /* shape outside what the kernels support       */
} pqk_status_t;

/* Stats slots written by the device entry points (int64 array of PQK_STATS_LEN). */
enum {
  PQK_STAT_UNIQUE_CENTERS = 0, /* distinct center codes after dedup                 */
  PQK_STAT_FLAGGED = 1,        /* codes the first-tier scan did not certify          */
  PQK_STAT_NNZ_TOTAL = 2,      /* sum of histogram support sizes over filled (k,m)  */
  PQK_STAT_EMPTY = 3,          /* empty clusters repaired                           */
  PQK_STAT_FILLED = 4,         /* clusters with >=1 member                          */
  PQK_STAT_VOTE_EXACT = 5,     /* (k,m) votes resolved by the double-double path    */
  PQK_STAT_ENCODE_FLAGGED = 6, /* encoder (vector,m) pairs recomputed in fp64       */
  PQK_STAT_NCHUNKS = 7,        /* center chunks streamed by the assignment scan     */
  PQK_STAT_VOTE_FP64 = 8,      /* (k,m) votes not certified by the fp32 filter      */
  PQK_STAT_FLAGGED_FP64 = 9,   /* codes decided by the exact fp64 rescan            */
  PQK_STAT_LOOKUP_BYTES = 10,  /* bytes per table lookup of the first-tier scan (2 or 4) */
  PQK_STATS_LEN = 24           /* slots 0..15 public, 16..23 scratch accumulators   */
};

/* ---- library / device info -------------------------------------------------- */
int pqk_abi_version(void);
const char* pqk_last_error(void); /* thread-local message of the last failure */
int pqk_device_info(int32_t device, int32_t* sm_count, int32_t* smem_optin_bytes);
int32_t pqk_padded_m(int32_t m); /* row stride of device code layout, 0 if unsupported */
int64_t pqk_launch_count(void);  /* kernels launched by this library since load */
/* Record the given cudaEvent_t handles (NULL to clear) immediately before and after
 * every assignment-scan kernel launch (benchmark roofline timing). */
int pqk_set_profile_events(void* before_scan, void* after_scan);

/* ---- host-side helpers (pure functions, no GPU) ------------------------------ */
/* Power-of-two exponent e such that ldexp(T, e) is representable in fp32 normal
 * range with headroom for M-term sums; *fp64_only = 1 when no such e exists
 * (then the assignment runs the exact fp64 scan for every code). */
int pqk_table_scale(const double* tables, int64_t count, int32_t* exp2_out, int32_t* fp64_only_out);

/* numpy pairwise-summation tree (numpy/_core/src/umath/loops_utils.h.src,
 * pairwise_sum, PW_BLOCKSIZE=128) used by np.mean in clustering.py:448-449.
 * Plan sizes, then the plan itself: leaves (offset,length) left-to-right, and per
 * depth d (0 = root) a node list (a,b): b<0 -> leaf a; else children a,b at d+1. */
int pqk_pairwise_plan_size(int64_t n, int64_t* nleaves, int32_t* ndepth, int64_t* nnodes);
int pqk_pairwise_plan_build(int64_t n, int64_t* leaf_off, int32_t* leaf_len,
                            int64_t* depth_start /* ndepth+1 */, int32_t* node_a, int32_t* node_b);

/* ---- device-pointer entry points (stream-ordered; stream is a cudaStream_t) -- */
/* T32[mp][l][l] = fl32(ldexp(T64[m][l][l], exp2)), zeros for pad subspaces. */
int pqk_tables_to_f32(const double* d_t64, int32_t m, int32_t l, int32_t exp2, float* d_t32, void* stream);

/* Pad (n, m) codes to the (n, MP) device layout. */
int pqk_pad_codes_device(const uint8_t* d_raw, int64_t n, int32_t m, uint8_t* d_padded, void* stream);

/* Nearest-center assignment (replaces _assign_linear_scan clustering.py:167-197 and
 * paired_distance_sq at clustering.py:447): labels[n] = argmin_k sum_m T[m][x_n^m][c_k^m]
 * in float64 ascending-m order with lowest index on ties, and sd_sq[n] the float64
 * distance to that center, bit-identical to the reference. */
size_t pqk_assign_workspace_bytes(int64_t n, int64_t k, int32_t m, int32_t l);
/* Scan tiers of pqk_assign_device.  Mode 0 (default): for problems of >= 2^31 lookups a
 * fixed-point first tier with exact integer sums, certified against the quantisation
 * error — 8-bit tables (1-byte lookups, the six smallest chunk keys per code) for padded
 * M = 4, 16-bit tables (2-byte lookups) for padded M 8 / 16 — then the fp32 scan over the
 * uncertified list when it is long (>= 256 codes per SM) and the exact fp64 rescan for
 * the rest.  Mode 1: the fp32 scan first.  Mode 2: the fixed-point tier at any size.
 * Mode 3: as 2 with the fp32 list tier for any list length.  Modes 4 / 5: as 2 / 3 with
 * the 16-bit tier also at padded M = 4.  Labels and sd_sq are identical in every mode
 * (process-wide setting, for A/B measurement and tests). */
int pqk_set_scan_mode(int32_t mode);
int32_t pqk_get_scan_mode(void);
int pqk_assign_device(const uint8_t* d_codes, int64_t n, int32_t m, int32_t l,
                      const uint8_t* d_centers, int64_t k,
                      const double* d_t64, const float* d_t32, int32_t fp64_only,
                      void* d_ws, size_t ws_bytes,
                      uint32_t* d_labels, double* d_sd_sq, int64_t* d_stats, void* stream);

/* sd[n] = sum_m T[m][a_n^m][b_{idx_n}^m] (float64, ascending m) — pq.py:271-290 with
 * b = centers[labels] (clustering.py:447).  idx may be NULL (b row-aligned with a). */
int pqk_paired_distance_device(const uint8_t* d_a, const uint8_t* d_b, const uint32_t* d_idx, int64_t n,
                               int32_t m, int32_t l, const double* d_t64, double* d_out, void* stream);

/* Histogram of member subindices (clustering.py:344-347) and counts (clustering.py:458):
 * hist[k][m][s] (uint32, zeroed here), counts[k] (uint32, zeroed here).  Shards of
 * up to 2^32 - 1 codes (the scan runs in 2^30-code windows); over all shards the
 * total stays below 2^32 so the reduced counts fit uint32. */
int pqk_histogram_device(const uint8_t* d_codes, int64_t n, int32_t m, int32_t l,
                         const uint32_t* d_labels, int64_t k, uint32_t* d_hist, uint32_t* d_counts, void* stream);

/* Sparse-voting update (clustering.py:349-356): for filled k,
 * new_centers[k][m] = argmin_j sum_s hist[k][m][s] * T[m][s][j] (lowest j on ties,
 * exact-arithmetic argmin: certified fp32 filter on d_t32 (nullable), then certified
 * fp64, double-double on near ties).  Empty clusters get code 0 (repaired by
 * pqk_repair_device).  Writes NNZ_TOTAL, FILLED, EMPTY, VOTE_EXACT stats.  Requires
 * hist/counts already reduced over all shards. */
int pqk_vote_device(const uint32_t* d_hist, const uint32_t* d_counts, int64_t k, int32_t m, int32_t l,
                    const double* d_t64, const float* d_t32, uint8_t* d_new_centers, int64_t* d_stats,
                    void* stream);

/* The same vote with the fp16 first-stage tables prebuilt once per table set
 * (pqk_vote_tables16_device: T16 = fp16(T32 * 2^f) per subspace, M*256*256 halves,
 * L = 256 only) instead of rebuilt on every call; d_t16 NULL = pqk_vote_device. */
int pqk_vote_tables16_device(const float* d_t32, int32_t m, int32_t l, void* d_t16, void* stream);
int pqk_vote16_device(const uint32_t* d_hist, const uint32_t* d_counts, int64_t k, int32_t m, int32_t l,
                      const double* d_t64, const float* d_t32, const void* d_t16, uint8_t* d_new_centers,
                      int64_t* d_stats, void* stream);

/* Empty-cluster repair (clustering.py:460-466): the E empty clusters (ascending k)
 * take the codes of the E codes with largest sd_sq (lowest index among ties).  Code
 * indices are 32-bit in the selection keys: n (and base_index + n) <= 2^32. */
size_t pqk_repair_workspace_bytes(int64_t n, int64_t k);
int pqk_repair_device(const double* d_sd_sq, const uint8_t* d_codes, int64_t n, int32_t m,
                      const uint32_t* d_counts, int64_t k, uint8_t* d_new_centers,
                      void* d_ws, size_t ws_bytes, int64_t* d_stats, void* stream);
/* Local top-E candidates for the multi-GPU repair: writes E (key,index) pairs
 * sorted by (sd_sq desc, index asc); index offset by base_index. */
int pqk_repair_candidates_device(const double* d_sd_sq, int64_t n, int64_t base_index, int64_t e,
                                 void* d_ws, size_t ws_bytes, uint64_t* d_out_keys, int64_t* d_out_index,
                                 void* stream);

/* Objective sums (clustering.py:448-449): out[0] = pairwise_sum(sqrt(sd)), out[1] =
 * pairwise_sum(sd) with numpy's exact tree (plan from pqk_pairwise_plan_build, uploaded). */
size_t pqk_objective_workspace_bytes(int64_t nleaves, int64_t nnodes);
int pqk_objective_device(const double* d_sd_sq, int64_t n, int64_t nleaves, int32_t ndepth,
                         const int64_t* d_leaf_off, const int32_t* d_leaf_len,
                         const int64_t* h_depth_start, const int32_t* d_node_a, const int32_t* d_node_b,
                         void* d_ws, size_t ws_bytes, double* d_out2, void* stream);

/* PQ encoder (pq.py:205-231): codes[n][m] = argmin_l sum_d (x - c_l)^2 in float64
 * sequential order (scipy cdist), lowest l on ties.  vectors (n, d) fp32,
 * codewords (m, l, d/m) fp32; code rows written with stride code_stride (pad bytes 0). */
int pqk_encode_device(const float* d_vectors, int64_t n, int32_t d, const float* d_codewords,
                      int32_t m, int32_t l, uint8_t* d_codes, int32_t code_stride,
                      int64_t* d_stats, void* stream);

/* Codebook training (pq.py:127-152, one Lloyd step of _lloyd_subspace on subspace
 * columns [col0, col0+dsub) of fp32 points (n, d)): labels, counts, per-(codeword, dim)
 * sums in point-index order, centers[filled] = sums / counts (fp64, in place), and —
 * only when some codeword is empty (count in d_stats[PQK_STAT_EMPTY]) — the
 * reference's `own` = np.sum((x - c[label])**2, axis=1) for the host-side reseed. */
size_t pqk_train_workspace_bytes(int64_t n, int32_t dsub);
int pqk_train_step_device(const float* d_x, int64_t n, int32_t d, int32_t col0, int32_t dsub, double* d_centers,
                          int32_t l, int32_t* d_labels, double* d_sums, int32_t* d_counts, double* d_own,
                          void* d_ws, size_t ws_bytes, int64_t* d_stats, void* stream);

/* DistanceTables (pq.py:254-268): tables[m][i][j] = sum_d (c_i - c_j)^2, float64 with the
 * difference and square rounded separately, summed in increasing d; codewords (m, l,
 * dsub) float32, tables (m, l, l) float64. */
int pqk_build_tables_device(const float* d_codewords, int32_t m, int32_t l, int32_t dsub, double* d_tables,
                            void* stream);

/* Original-space evaluation (baselines.py:26-37 cluster_means, :385-413
 * original_space_error).  means[k][:] = float64 mean of the rows labelled k, summed in
 * increasing row index from 0.0 (np.bincount with weights), 0 for empty clusters;
 * counts[k] optional.  x is (n, d) row-major, dtype 0 = float32, 1 = float64; labels in
 * [0, k), n < 2^32. */
size_t pqk_cluster_means_workspace_bytes(int64_t n, int32_t k);
int pqk_cluster_means_device(const void* d_x, int32_t dtype, int64_t n, int32_t d, const int32_t* d_labels,
                             int32_t k, double* d_means, int32_t* d_counts, void* d_ws, size_t ws_bytes,
                             void* stream);
/* sq[i] = np.sum((x[i] - centers[labels[i]])**2): float64, numpy's pairwise order over d.
 * original_space_error = mean(sqrt(sq)) via pqk_objective_device. */
int pqk_assigned_sq_device(const void* d_x, int32_t dtype, int64_t n, int32_t d, const double* d_centers,
                           const int32_t* d_labels, double* d_sq, void* stream);

/* Bk-means baseline (baselines.py:229-382).  Packed codes are MSB-first bytes
 * (np.packbits) in rows padded to wp in {4, 8, 16, 32} bytes (zero pad bytes).
 * binarize: bit b = (x . R[:, b] >= 0), R float64 (d, bits) with orthonormal columns;
 *   fp32 filter with a rigorous bound, exact double-double sign for the rest (count in
 *   d_stats[PQK_STAT_ENCODE_FLAGGED]).
 * hamming_assign: labels = argmin_k popcount(code ^ center_k), lowest k on ties; sd =
 *   dist^2 (float64, nullable) and dist (nullable).  k <= 2^24.
 * hamming_matrix: out[i][k] = popcount(code_i ^ center_k) (hamming_to_centers).
 * majority_update: counts, per-bit ones, new_centers[k] = packbits(2*ones > count) for
 *   filled k (0 for empty), EMPTY/FILLED stats; then pqk_repair_device(sd, ...) with
 *   m = wp repairs the empty clusters. */
int pqk_binarize_device(const float* d_x, int64_t n, int32_t d, const double* d_rotation, int32_t bits,
                        uint8_t* d_codes, int32_t code_stride, int64_t* d_stats, void* stream);
int pqk_hamming_assign_device(const uint8_t* d_codes, int64_t n, int32_t wp, const uint8_t* d_centers, int64_t k,
                              uint32_t* d_labels, double* d_sd, int32_t* d_dist, void* stream);
int pqk_hamming_matrix_device(const uint8_t* d_codes, int64_t n, int32_t wp, const uint8_t* d_centers, int64_t k,
                              int32_t* d_out, void* stream);
int pqk_majority_update_device(const uint8_t* d_codes, int64_t n, int32_t wp, int32_t bits, const uint32_t* d_labels,
                               int64_t k, int32_t* d_counts, int32_t* d_ones, uint8_t* d_new_centers,
                               int64_t* d_stats, void* stream);

/* File ingest for the streaming pipeline (io.py formats).  unpack_vecs: n raw
 * fvecs (itemsize 4) / bvecs (itemsize 1) records -> dense float32 rows; err[0] = first
 * record (base_record + r) whose int32 dimension != dim (UINT64_MAX if none; callers
 * initialise it), err[1] = that dimension.  unpack_codes: n x m PQKC payload bytes ->
 * rows of `stride` bytes (pad 0); err[0] = first byte position (record * m + column)
 * holding a subindex >= l, err[1] = its value.  d_raw of unpack_vecs must be 4-byte
 * aligned for itemsize 4. */
int pqk_unpack_vecs_device(const uint8_t* d_raw, int64_t n, int32_t dim, int32_t itemsize, int64_t base_record,
                           float* d_out, uint64_t* d_err, void* stream);
int pqk_unpack_codes_device(const uint8_t* d_raw, int64_t n, int32_t m, int32_t l, int64_t base_record,
                            uint8_t* d_out, int32_t stride, uint64_t* d_err, void* stream);

/* ---- host-buffer entry points (the reference-facing plugin boundary) ---------- */
/* AssignStrategy (clustering.py:200): labels (and optionally sd_sq) for host codes. */
int pqk_assign_host(const uint8_t* codes, int64_t n, int32_t m, const uint8_t* centers, int64_t k,
                    const double* tables, int32_t l, uint32_t* labels, double* sd_sq /* nullable */,
                    int32_t device);
/* encode (pq.py:205): vectors (n,d) fp32 host, codewords (m,l,d/m) fp32 host -> codes (n,m) */
int pqk_encode_host(const float* vectors, int64_t n, int32_t d, const float* codewords, int32_t m,
                    int32_t l, uint8_t* codes, int32_t device);
/* One Lloyd iteration of fit (clustering.py:443-466) on host buffers: assign,
 * objective sums, histogram, sparse vote, repair.  Outputs labels (n), new centers
 * (k,m), obj2[2] = {sum sqrt(sd), sum sd} and stats (PQK_STATS_LEN). */
int pqk_lloyd_step_host(const uint8_t* codes, int64_t n, int32_t m, const uint8_t* centers, int64_t k,
                        const double* tables, int32_t l, uint32_t* labels, uint8_t* new_centers,
                        double* obj2, int64_t* stats, int32_t device);
/* Release the cached per-device context of the host entry points. */
int pqk_host_release(int32_t device);

/* ---- single-process multi-GPU exchange (peer memory over NVLink/NVSwitch) ------- */
/* d_out[i] = sum over g of peer_ptrs[j][i], i < count (uint32; peer_ptrs is a HOST array
 * of g <= 16 device pointers, any device with peer access enabled; d_out may alias one of
 * them).  The histogram/count allreduce of a sharded iteration (clustering.py:344-347,
 * :458) as a reduce-scatter: each device sums its slice of clusters from every peer. */
int pqk_peer_sum_device(const uint32_t* const* peer_ptrs, int32_t g, int64_t count, uint32_t* d_out, void* stream);
/* cudaDeviceEnablePeerAccess for every ordered pair of distinct listed devices. */
int pqk_enable_peer_access(const int32_t* devices, int32_t g);

/* ---- diagnostics -------------------------------------------------------------- */
/* tcgen05 self-test: C (128 x 256, fp32) = A (128 x k, fp16, row-major) * B (256 x k,
 * fp16, row-major)^T through UMMA descriptors, TMEM and tcgen05.ld (k % 16 == 0). */
int pqk_tc_selftest(const void* d_a_f16, const void* d_b_f16, float* d_c, int32_t k, void* stream);
/* Measured shared-memory load ceiling (bench roofline denominator): conflict-free
 * LDS.128 from one 1024-thread CTA per SM over `iters` x 16 loads per thread; returns
 * bytes/s (and the timed launch in ms) measured with CUDA events on `stream`. */
int pqk_smem_probe(int32_t device, int32_t iters, double* bytes_per_s, double* ms_out, void* stream);
/* Tensor-memory read bandwidth (tcgen05.ld, all 512 columns of one CTA per SM, 16 warps):
 * the ceiling of the encoder's epilogue.  Bytes/s of the whole GPU, best of 3. */
int pqk_tmem_probe(int32_t device, int32_t iters, double* bytes_per_s, double* ms_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PQK_B200_H */
