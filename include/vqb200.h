/*
 * vqb200.h -- C ABI of libvqb200.so, the B200 (sm_100a) LBG vector
 * quantisation hot path.  Drop-in for the reference arxiv/paper_0910_4711
 * (package vqkit, pure Python + numba).
 *
 * The reference has no C ABI: its drop-in seam is the module object
 * vqkit._kernels, which every caller looks up by attribute at call time
 * (core.py:20,244,258,271,315-316,338,380,392-393,402,421-422;
 * parallel.py:22,114,121,190,273,290,316,321; codec.py:11,89,154-155).
 * Two surfaces are exported:
 *
 *  1. Kernel surface (stateless, HOST buffers, same argument meaning as
 *     vqkit._kernels): vqb_assign_range, vqb_update_rows, vqb_column_sums,
 *     vqb_sum_inorder, vqb_pair_distance.  A ctypes shim can rebind the
 *     reference's _kernels attributes to these.
 *
 *  2. Session surface (device-resident training set): vqb_open / vqb_train /
 *     vqb_assign / vqb_update / vqb_close, replacing the reference's entry
 *     points lbg_train (core.py:366-430), parallel_lbg_train
 *     (parallel.py:256-329), assign_cells (core.py:292-316), update_codebook
 *     (core.py:319-339) and encode (codec.py:62-93) without moving the
 *     training set over PCIe on every pass.  The vqb_step_* calls expose one
 *     Lloyd pass at a time for the multi-GPU loop (one process per GPU, the
 *     caller allreduces the packed int64 exchange buffer over NCCL).
 *
 * Conventions.
 *  - Status codes mirror the reference's exception hierarchy (errors.py:8-29):
 *    0 ok, 1 UsageError, 2 ConfigError, 3 DomainError, 4 InternalError
 *    (CUDA failures included), 5 FormatError.  vqb_last_error() returns the message of the
 *    calling thread's last failure.
 *  - Host buffers are caller-owned; device memory is owned by the session.
 *  - Every call is synchronous on return unless its name says `step` / `async`.
 *  - Metric codes: 0 squared_euclidean, 1 euclidean (_kernels.py:14-15).
 *  - No CPU fallback: without a CUDA device every compute call returns 4.
 */
#ifndef VQB200_H
#define VQB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VQB_OK 0
#define VQB_USAGE 1
#define VQB_CONFIG 2
#define VQB_DOMAIN 3
#define VQB_INTERNAL 4
#define VQB_FORMAT 5 /* FormatError (errors.py:24-25): corrupt stream / payload */

const char* vqb_last_error(void);
int vqb_version(void);
int vqb_device_count(int* count);

/* ---- kernel surface: replaces vqkit._kernels (_kernels.py:18-98) ---- */

/* _kernels.assign_range (_kernels.py:18-36): rows [start, stop) of
 * vectors[m][dim] against codebook[size][dim]; writes out_cells[z] (int64)
 * and out_dists[z] (FP64, sqrt'ed under metric 1) for z in [start, stop). */
int vqb_assign_range(const double* vectors, int64_t m, int64_t dim, const double* codebook,
                     int64_t size, int64_t start, int64_t stop, int metric,
                     int64_t* out_cells, double* out_dists);

/* _kernels.update_rows (_kernels.py:39-66): centroids of codevector rows
 * i with i % stride == worker; empty rows copy old_codebook.  Other rows of
 * out_codebook / out_counts are left untouched. */
int vqb_update_rows(const double* vectors, int64_t m, int64_t dim, const int64_t* cells,
                    const double* old_codebook, int64_t size, int64_t worker, int64_t stride,
                    double* out_codebook, int64_t* out_counts);

/* _kernels.column_sums (_kernels.py:81-89), ascending row order. */
int vqb_column_sums(const double* vectors, int64_t m, int64_t dim, double* out);

/* _kernels.sum_inorder (_kernels.py:92-98), strict left-to-right. */
int vqb_sum_inorder(const double* values, int64_t n, double* out);

/* core.split_codebook (core.py:277-289): out[2*size][dim], rows 2i = c_i +
 * delta and 2i+1 = c_i - delta (one rounding each); VQB_CONFIG unless
 * delta > 0. */
int vqb_split_codebook(const double* codebook, int64_t size, int64_t dim, double delta, int device,
                       double* out);

/* _kernels.pair_distance (_kernels.py:69-78). */
int vqb_pair_distance(const double* a, const double* b, int64_t dim, int metric, double* out);

/* ---- session surface ---- */

typedef struct vqb_session vqb_session;

/* Training set upload (TrainingSet, core.py:72-99).  Exactly one of x32 / x64
 * is non-null.  float32 rows (exact in FP64, core.py:47-60) take the FP32
 * candidate path; float64 rows take the exact-FP64 path.  `rows`/`dim` are
 * this process's shard; row_offset / n_global place it in the global set
 * (n_global = rows, row_offset = 0 for one GPU).  device = CUDA ordinal. */
int vqb_open(const float* x32, const double* x64, int64_t rows, int64_t dim, int64_t row_offset,
             int64_t n_global, int device, vqb_session** out);
int vqb_close(vqb_session* s);
/* Use a caller stream (cudaStream_t as void*), e.g. torch's current stream. */
int vqb_set_stream(vqb_session* s, void* stream);
/* max |x| over this shard (+inf when any value is non-finite). */
int vqb_local_maxabs(vqb_session* s, double* out);
/* Per-column stats of this shard's rows: colmax[dim] = max |x| (+inf when a
 * value is non-finite), collow[dim] = exponent of the lowest set bit
 * (INT32_MAX for a column of zeros).  Ranks combine them (MAX / MIN) into the
 * global stats that fix the two-word fixed-point plan of the cell sums
 * (vqb_train_config.global_colmax / global_collow). */
int vqb_local_colstats(vqb_session* s, double* colmax, int32_t* collow);
/* info[5] = {candidate pass on (FP32 / tensor-core fast path), candidate
 * width (16/32/64, rows zero-padded; 0: L > 64, FP64 scan only), rows held as
 * float64 (not float32-exact), cell sums exact on the two-word grid, the
 * reference's own FP64 cell sums provably exact}. */
int vqb_session_info(vqb_session* s, int32_t* info);

typedef struct {
  int64_t target_size;               /* LbgConfig.target_size (power of two) */
  double epsilon;                    /* relative-drop threshold, <= test */
  double delta;                      /* additive split offset */
  int64_t max_iterations_per_level;  /* guard (warning, not error) */
  int32_t metric;                    /* 0 squared_euclidean, 1 euclidean */
  int32_t ordered;                   /* -1 auto, 0 two-word fixed-point sums, 1 reference order */
  const double* global_colmax;       /* [dim] or NULL: this shard's column stats */
  const int32_t* global_collow;      /* [dim] or NULL */
} vqb_train_config;

typedef struct {
  int64_t codebook_size;
  int64_t iteration;
  double td;
  int64_t empty_cells;
  double seconds;
} vqb_level_iteration; /* LevelIteration (core.py:162-172) */

typedef struct {
  double total;
  int64_t n_hist;
  int64_t n_warn;
  int64_t passes;
  int64_t flagged_rows;  /* rows re-ranked in FP64 over the run */
  int64_t evals;         /* sum over passes of rows * codebook size (this shard) */
  int64_t final_size;
  int32_t fast_path;     /* 1: FP32 candidate + FP64 re-rank; 0: exact FP64 scan */
  int32_t ordered;
  int64_t flagged_full;  /* of flagged_rows, those whose shortlist overflowed (full FP64 scan) */
  int32_t sums_exact;    /* 1: every coordinate is exact on the two-word fixed-point grid */
  int32_t ref_exact;     /* 1: the reference's own FP64 cell sums are provably exact too (so the
                            fixed-point centroids equal update_rows' bit for bit) */
} vqb_train_summary;

/* Full LBG design on the device (lbg_train / parallel_lbg_train).  Outputs:
 * codebook_out[target_size][dim], hist[hist_cap] (nullable: fetch the whole
 * history afterwards with vqb_step_history, sized from summary->n_hist),
 * warn_sizes[warn_cap] (level sizes whose guard tripped), final_dists[rows]
 * (nullable: distances of the last allocation pass, for
 * DistortionStats.per_worker). */
int vqb_train(vqb_session* s, const vqb_train_config* cfg, double* codebook_out,
              vqb_level_iteration* hist, int64_t hist_cap, int64_t* warn_sizes, int64_t warn_cap,
              double* final_dists, vqb_train_summary* summary);

/* Allocation with a fixed codebook (assign_cells / encode) over this shard.
 * cells64 / idx32 / dists are nullable; total = deterministic tree-order sum. */
int vqb_assign(vqb_session* s, const double* codebook, int64_t size, int metric, int64_t* cells64,
               uint32_t* idx32, double* dists, double* total);

/* Centroid update for a given cell table (update_codebook / parallel_update). */
int vqb_update(vqb_session* s, const int64_t* cells, const double* old_codebook, int64_t size,
               double* new_codebook, int64_t* counts, int64_t* n_empty);

/* ---- step API for the multi-GPU loop (one process per GPU) ----
 * begin: uploads config, enqueues the local column-sum pass.
 * Each pass: step_local (assign + re-rank + epilogue) ; caller allreduces the
 * exchange buffer (int64 SUM) on the session stream ; step_finalize.
 * The first finalize after begin computes the global centroid.
 * step_poll reports done (synchronises the stream). */
int vqb_step_begin(vqb_session* s, const vqb_train_config* cfg);
int vqb_step_local(vqb_session* s);
int vqb_step_finalize(vqb_session* s);
int vqb_step_exchange(vqb_session* s, int64_t** device_words, int64_t* count);
int vqb_step_poll(vqb_session* s, int* done);
int vqb_step_result(vqb_session* s, double* codebook_out, vqb_level_iteration* hist,
                    int64_t hist_cap, int64_t* warn_sizes, int64_t warn_cap, double* final_dists,
                    vqb_train_summary* summary);
/* The last finished run's history (DistortionStats.history, core.py:175-197):
 * up to cap records into hist, *count = records recorded. */
int vqb_step_history(vqb_session* s, vqb_level_iteration* hist, int64_t cap, int64_t* count);

/* Fixed-size Lloyd passes over shards (the multi-GPU form of
 * vqb_lloyd_step_f32): begin uploads the codebook and fixes the common
 * fixed-point plan (global column stats; NULL: this shard's); per pass
 * vqb_lloyd_local (assign + re-rank + distortion + cell sums), the caller
 * allreduces vqb_step_exchange's int64 buffer (SUM), then vqb_step_finalize
 * makes the centroids of the combined sums current on every rank (same bits
 * everywhere: integer sums). vqb_step_result reads the codebook back. */
int vqb_lloyd_begin(vqb_session* s, const double* codebook, int64_t size, const double* global_colmax,
                    const int32_t* global_collow);
int vqb_lloyd_local(vqb_session* s);

/* ---- one-shot host-buffer calls (end-to-end path, copies included) ---- */

/* encode (codec.py:62-93) of host float32 rows: pipelined H2D / assign / D2H
 * in row chunks; idx_out uint32[n]; total (nullable) = tree-order distortion. */
int vqb_encode_f32(const float* x, int64_t n, int64_t dim, const double* codebook, int64_t size,
                   int device, uint32_t* idx_out, double* total);

/* One Lloyd iteration from host buffers (assign + distortion + update): the
 * kernel-surface round trip a reference caller makes per pass
 * (core.py:392-406).  Outputs new_codebook[size][dim], td (tree order),
 * n_empty; cells_out (nullable, int64[n]). */
int vqb_lloyd_step_f32(const float* x, int64_t n, int64_t dim, const double* codebook,
                       int64_t size, int device, double* new_codebook, int64_t* cells_out,
                       double* td, int64_t* n_empty);

/* ---- data formats either side of the path ----
 * Stateless, host buffers, synchronous.  `images` stacked uint8 rasters
 * [images][height][width]; their block vectors are image-major, each image's
 * ceil(h/b) x ceil(w/b) blocks row-major, each block row-major (b*b values). */

/* storage.pixels_to_blocks (storage.py:281-293) / image_to_blocks
 * (storage.py:274-278): ragged edges replicated (np.pad mode "edge").
 * Exactly one of out64 (float64, the reference's dtype) / out32 is non-null. */
int vqb_pixels_to_blocks(const uint8_t* pixels, int64_t images, int64_t height, int64_t width,
                         int64_t block, int device, double* out64, float* out32);

/* storage.blocks_to_image raster (storage.py:296-311): clamp to [0, 255],
 * floor(v + 0.5), crop the padding (NaN -> 0). */
int vqb_blocks_to_pixels(const double* vectors, int64_t images, int64_t height, int64_t width,
                         int64_t block, int device, uint8_t* pixels);

/* codec.decode (codec.py:96-114): out[j][:] = codebook[indices[j]][:];
 * VQB_FORMAT when an index >= size. */
int vqb_decode(const uint32_t* indices, int64_t n, const double* codebook, int64_t size, int64_t dim,
               int device, double* out);

/* decode fused with blocks_to_image: the block indices of `images` images ->
 * pixels, without the float64 block matrix (cli.py decode of an image). */
int vqb_decode_pixels(const uint32_t* indices, int64_t images, int64_t height, int64_t width,
                      int64_t block, const double* codebook, int64_t size, int device, uint8_t* pixels);

/* codec.reconstruction_distortion (codec.py:135-156): per-row pair_distance
 * (_kernels.py:69-78) in the reference arithmetic; total summed in input
 * order (sum_inorder) for n <= 2^20 rows, else per-2048-row fixed tree +
 * in-order over tiles. */
int vqb_reconstruction_distortion(const double* a, const double* b, int64_t n, int64_t dim, int metric,
                                  int device, double* total);

/* The session's float32 rows back to the host (out[rows][dim]); VQB_USAGE for
 * a session that holds float64 rows.  A pixel-fed TrainingSet materialises
 * its float64 field from this on first access. */
int vqb_rows_f32(vqb_session* s, float* out);

/* Session over the block vectors of `images` uint8 images, vectorised on the
 * device (1 byte per sample over PCIe instead of the reference's float64
 * copy, core.py:47-60): the training set of image_to_blocks + TrainingSet. */
int vqb_open_pixels(const uint8_t* pixels, int64_t images, int64_t height, int64_t width, int64_t block,
                    int device, vqb_session** out);

/* Session over `rows` rows of an isotropic Gaussian mixture drawn on the
 * device (replaces the host generators behind the benchmark training sets,
 * reference bench.py:59-62 / SURVEY 8(f) row 1; no row crosses PCIe).
 * Component c has mean means[c][dim] and standard deviation sigmas[c]; it is
 * picked uniformly, or as the first c with u < cum_weights[c] when the
 * (nondecreasing, ending at 1) cumulative weights are given.  Row g (global
 * index row_offset + r) draws from Philox4x32-10 with counter (g, call) and
 * key `seed`, so a shard [row_offset, row_offset + rows) of n_global rows is
 * the same slice of the same set on any device count.  Every bit is
 * reproducible on the host (oracle/vq_oracle.c vq_gmm_rows). */
int vqb_open_gmm(const float* means, const float* sigmas, const double* cum_weights, int64_t components,
                 int64_t rows, int64_t dim, int64_t row_offset, int64_t n_global, uint64_t seed, int device,
                 vqb_session** out);

/* Device-resident timing of one imaging kernel (0 pixels_to_blocks f32,
 * 1 pixels_to_blocks f64, 2 blocks_to_pixels, 3 decode, 4 decode_pixels,
 * 5 per-row pair distances): mean ms per launch over `reps` and the
 * algorithmic bytes of one launch (bench.py --workload formats). */
int vqb_bench_formats(int which, int64_t images, int64_t height, int64_t width, int64_t block, int64_t n,
                      int64_t dim, int64_t size, int reps, double* ms_out, double* bytes_out);

/* ---- host helpers of the Python types (TrainingSet, core.py:72-99) ---- */

/* memcpy split over host threads (the TrainingSet snapshot of float32 rows). */
int vqb_host_copy(void* dst, const void* src, int64_t bytes);

/* Index of the first inf / NaN among n float32 values, or -1 (host threads);
 * TrainingSet's "training vector i component j is not finite" check. */
int vqb_first_nonfinite_f32(const float* x, int64_t n, int64_t* first);
int vqb_first_nonfinite_f64(const double* x, int64_t n, int64_t* first);

/* Pipe microbenchmark (0 FFMA, 1 FFMA2, 2 FFMA+top-2 mix, 3 DADD): lane-ops/s. */
int vqb_pipe_microbench(int which, int blocks_per_sm, int iters, double* ops_per_s,
                        double* seconds);

/* Time `reps` device-resident Lloyd passes (assign + re-rank + update) at a
 * codebook (the bench's kernel-only step; each pass continues from the
 * previous update).  ms_segments[5] = average ms of [state reset (the codebook
 * staging happens in apply), assign, re-rank, epilogue, finalize+apply]; flagged = rows re-ranked
 * per pass. */
int vqb_bench_iteration(vqb_session* s, const double* codebook, int64_t size, int reps,
                        double* ms_segments, int64_t* flagged);

/* Time `reps` device-resident allocation passes (assign + re-rank + exact
 * distances + distortion) at a fixed codebook: ms_out = average ms per pass,
 * total_out = that pass's distortion, flagged = rows re-ranked per pass. */
int vqb_bench_assign(vqb_session* s, const double* codebook, int64_t size, int reps,
                     double* ms_out, double* total_out, int64_t* flagged);

/* Tensor-core candidate-pass probe (tests): raw fp32 accumulators of rows
 * [0,128) of the session against `codebook` (size a multiple of 256),
 * dump[128][size]; scales[5] = {ey, ew, kn, tc_on, tc_bad}. */
int vqb_debug_tc_tile(vqb_session* s, const double* codebook, int64_t size, float* dump,
                      int32_t* scales);

/* Host->device copy-engine bandwidth probe: mode 0 staged/pinned upload,
 * 1 plain cudaMemcpy, 2 cudaHostRegister + upload (register cost included). */
int vqb_bench_upload(const void* src, int64_t bytes, int mode, double* seconds);

#ifdef __cplusplus
}
#endif

#endif /* VQB200_H */
