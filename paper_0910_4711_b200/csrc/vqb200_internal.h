// Internal declarations shared by the kernels (kernels.cu) and the C-ABI /
// native training loop (api.cu).  Not part of the public ABI: that is
// include/vqb200.h.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "refarith.cuh"

namespace vqb {

constexpr int kHistRing = 8192;  // device ring of history records, drained by the host per batch
constexpr int kMaxWarn = 64;     // one warning per level at most
constexpr int kTdTile = 2048;    // rows per distortion partial (fixed, global)
constexpr int kEpiThreads = 1024; // dist/TD block: 2 rows per thread per 2048-row tile

// metric codes (reference _kernels.py:14-15)
constexpr int kSquared = 0;
constexpr int kEuclidean = 1;

// device loop modes
constexpr int kModeTrain = 0;       // split + Lloyd loop (core.py:384-415)
constexpr int kModeFinalAssign = 1; // target_size == 1 (core.py:417-422)
constexpr int kModeAssignOnly = 2;  // assign_cells / encode with a fixed codebook
constexpr int kModeUpdateOnly = 3;  // update_codebook for a given cell table
constexpr int kModeLloydStep = 4;   // one assign + update pass, no convergence logic

struct HistRec {
  int size;
  int iteration;
  double td;
  long long empty;
  unsigned long long t_ns;
};

// Loop state, resident on the device; every kernel of a pass reads it so the
// host never needs to know the current codebook size (passes can be enqueued
// speculatively and early-exit once `done` is set).
struct DevState {
  // configuration
  int target;
  int max_iter;
  int metric;
  int lo_shift;        // t: the low word of a two-word fixed-point value has 2^-(s_l + t) units
  int sums_exact;      // 1: every coordinate is exact on its column's two-word grid
  int ref_exact;       // 1: the reference's own FP64 cell sums are provably exact too
  double eps;
  double delta;
  long long n_global;  // rows over all shards (for the centroid of size 1)
  int mode;
  int ordered;         // 1: reference-order update/TD kernels (bit-identical, slow)
  // progress
  int size;
  int iteration;
  int done;
  int n_hist;          // records written so far (adjacent to done: one 8-byte poll reads both)
  int cur;             // which codebook buffer holds the current codebook
  double td_prev;
  double total;
  double last_td;
  long long last_empty;
  int n_warn;
  int warn_sizes[kMaxWarn];
  int flag_count;      // rows queued for the re-rank this pass (assign_fast -> shortlist)
  int flag2_count;     // rows whose shortlist overflowed -> full FP64 scan
  unsigned int cmax_bits;  // float bits of max_j ||c~_j|| (centred FP32 codebook)
  int passes;          // allocation passes executed
  int slabs;           // per-block cell-sum slabs the sums kernel of this pass wrote
  int skip;            // 1: the fused small-codebook pass did this whole pass (the per-kernel path idles)
  unsigned bar_count;  // grid barrier of the fused pass (arrivals, generation)
  unsigned bar_gen;
  int nonfinite;       // set_shift saw a non-finite |x| (host-buffer Lloyd step)
  // tensor-core candidate pass (assign_tc.cu): power-of-two scales of the
  // fp16 hi/lo operand split, chosen on the host from |x| / codebook bounds
  int tc_on;           // 1: the TC pass may run when tc_kmin <= size <= tc_kmax
  int tc_kmin, tc_kmax;
  int tc_ey, tc_ew, tc_kn;
  int tc_bad;          // staging saw an fp16-unrepresentable codebook value
  long long flagged_total;  // rows re-ranked over the whole run (diagnostic)
  long long flagged2_total; // of which needed the full FP64 scan
  long long evals;     // sum over passes of rows * size (this shard)
  int act;             // apply_kernel action bits (update 1, split 2)
  int act_src;         // buffer holding the source codebook of the action
  int act_k;           // source codebook size
  unsigned long long t0_ns;  // %globaltimer at the initial centroid
  // incremental cell sums (training loop): the codebook size the running sums
  // `acc` and the previous cells `idx_prev` describe (0: none), and the rows
  // whose cell changed this pass (the moved list)
  int acc_size;
  int nmoved;
  int hist_cap;        // ring capacity: record i lives in hist[i % hist_cap]
  HistRec* hist;       // device ring, session-owned; the host drains it as passes complete
};

// Packed exchange buffer (int64 words), one allreduce per pass in the
// multi-GPU loop: [hi sums K*L | counts K | td tile partials (FP64 bit
// patterns, zero on tiles another rank owns) | lo sums K*L].  A cell sum is
// the two-word fixed-point integer hi * 2^t + lo in units of 2^-(s_l + t)
// (per-column shift s_l, common t; see fixed_plan).
struct Exchange {
  long long* base;
  long long kmax;
  long long dim;
  long long ntiles;
  __host__ __device__ long long* sums() const { return base; }
  __host__ __device__ long long* counts() const { return base + kmax * dim; }
  __host__ __device__ long long* td() const { return base + kmax * dim + kmax; }
  __host__ __device__ long long* lo() const { return base + kmax * dim + kmax + ntiles; }
  __host__ __device__ long long words() const { return 2 * kmax * dim + kmax + ntiles; }
};

// ---- two-word fixed-point cell sums (the centroid numerators) ----
// Column l is scaled by 2^s_l with s_l = 61 - e_n - e_l (rows < 2^e_n,
// max |x_l| < 2^e_l), so the high words of n rows cannot overflow int64.  A
// coordinate x splits EXACTLY as x * 2^s_l = hi + lo * 2^-t (hi = the integer
// part of the magnitude, lo its remainder in units of 2^-t, t = 62 - e_n):
// exact whenever x has no set bit below 2^-(s_l + t) = 2^(2 e_n + e_l - 123)
// (at N = 2^20 and |x| < 512: every float32 |x| >= 2^-50), which is checked
// up front (colstats: the lowest set bit of every column; otherwise the
// reference-order path runs).  Integer
// sums commute, so the result is the exact cell sum -- deterministic,
// grid-independent and identical for every GPU count -- rounded once when it
// becomes a centroid.  When the reference's own ascending-order FP64 sum is
// exact as well (ref_exact: e_n + e_l - lowbit_l <= 53), the centroids are
// bit-identical to the reference's.
__host__ __device__ inline int ceil_log2_rows(long long n) {
  int e = 0;
  while (e < 62 && (1LL << e) < n) ++e;
  return e;
}
struct FixedCol {
  int s;          // column shift
  int exact;      // two-word split exact for every coordinate of the column
  int ref_exact;  // the reference's FP64 sums of this column are exact in any order
};
__host__ __device__ inline FixedCol fixed_plan(long long n_global, double maxabs, int minlow) {
  FixedCol f;
  const int e_n = ceil_log2_rows(n_global);
  const int t = 62 - e_n;
  int e_x = 0;
  if (maxabs > 0 && maxabs <= 1.7976931348623157e308) frexp(maxabs, &e_x);
  int s = 61 - e_n - e_x;
  s = s > 960 ? 960 : (s < -1020 ? -1020 : s);
  const bool zero = minlow == 0x7fffffff;  // column of zeros
  f.s = s;
  f.exact = (maxabs <= 1.7976931348623157e308) && (zero || (minlow + s + t >= 0 && s + t <= 1020));
  f.ref_exact = f.exact && (zero || e_n + e_x - minlow <= 53);
  return f;
}
__host__ __device__ inline int fixed_lo_shift(long long n_global) { return 62 - ceil_log2_rows(n_global); }

struct KernelArgs {
  // training data (this shard): exactly one of x32/x64 is non-null (x64 only
  // for float64 rows float32 cannot hold); dim = L
  const float* x32;
  const double* x64;
  // candidate rows of the FP32 / tensor-core passes: the rows rounded to
  // float32 and zero-padded to cdim in {16, 32, 64} (== x32 when L is one of
  // those and the rows are float32); rin[row] (nullable) bounds the rounding
  // ||x - fl32(x)|| <= 2^-24 ||x|| of float64 rows, widening the certified band
  const float* xc;
  int cdim;
  const float* rin;
  long long n;          // local rows
  long long n_global;   // rows over all shards (fixed-point plan)
  long long r0, r1;     // row range of the candidate pass (a chunk of [0, n))
  int dim;
  long long tile0;      // global index of this shard's first TD tile
  const float* mu;      // centring vector (FP32, dim)
  const int* cshift;    // per-column fixed-point shifts s_l (dim)
  // codebooks
  double* cb[2];        // FP64 master, double buffered, kmax x dim
  float* w;             // -2 * c~ (FP32), kpad x dim
  unsigned short* tcb;  // fp16 hi/lo operand image of the codebook for the TC pass (nullable)
  // fp16 hi/lo operand image of the resident rows (nullable; build_row_image):
  // per 128-row tile [yh 128 x L | yl 128 x L] in the smem layout, and
  // ||y~||^2 per row (-1: a row fp16 cannot hold)
  const unsigned short* aimg;
  const float* aq;
  float* nrm;           // ||c~||^2 (FP32), kpad
  long long kmax;
  // per-row outputs
  int* idx;
  int* flags;
  float* flag_thr;      // per queued row: band threshold m1 + 3E (FP32 expanded form)
  int* flags2;          // shortlist overflow rows
  double* dists;        // nullable
  Exchange ex;
  long long* partials;  // per-block fixed-point slabs, sms x (kmax*dim + kmax)
  double* ord;          // reference-order centroids (ordered mode), kmax x dim
  int* operm;           // ordered mode: rows sorted by cell, ascending within a cell (n)
  int* obase;           // ordered mode: per (cell, row block) offsets, kmax x oblocks
  int* oscan;           // ordered mode: scan scratch
  int oblocks;          // ordered mode: row blocks of the counting sort
  // incremental cell sums of the training loop (nullable: every pass sums all
  // rows): the previous pass's cells, the moved list [row | old cell | new
  // cell] (3 x mv_cap ints), this shard's running two-word sums
  // [hi kmax*dim | counts kmax | lo kmax*dim], and the moved-row count up to
  // which a pass updates them instead of summing every row again
  int* idx_prev;
  int* mv;
  long long mv_cap;
  long long* acc;
  long long delta_max;
  int diff_on;          // FFMA pass at L >= 32, K < 64: difference-form candidate values (VQB_DIFF=0: expanded)
  int small_on;         // candidate pass: assign_small_kernel takes K < 64 (VQB_SMALL=0: assign_fast_kernel does)
  DevState* st;
};

// Incremental cell sums.  Integer fixed-point sums are exact, so a pass may
// update the previous pass's sums by the rows that changed cell (+x into the
// new cell, -x out of the old one) and get the very words a full pass over
// every row would: late passes of a level move a few percent of the rows.
// delta_track: this pass keeps idx_prev / acc current; delta_go: it also
// takes the incremental path (acc describes this codebook size and few
// enough rows moved) -- read by every sums kernel of the pass after
// moved_scan_kernel has counted, so they all agree.
__device__ __forceinline__ bool delta_track(const KernelArgs& a, const DevState* st) {
  return a.acc != nullptr && st->mode == kModeTrain && !st->ordered;
}
__device__ __forceinline__ bool delta_go(const KernelArgs& a, const DevState* st) {
  return delta_track(a, st) && st->acc_size == st->size && (long long)st->nmoved <= a.delta_max;
}

// The reference's distance (_kernels.py:25-29) of row `row` to codevector j
// (FP64 master codebook cb), from the rows the reference sees: the float64
// rows when the session holds them, else the float32 rows (vectorised when L
// is the candidate width W).
template <int W>
__device__ __forceinline__ double row_dist(const KernelArgs& a, long long row, const double* cb, long long j) {
  if (a.x64) return ref_dist(a.x64 + row * a.dim, cb + j * a.dim, a.dim);
  if (a.dim == W) return winner_dist<float, W>(a.x32 + row * W, cb + j * W, W);
  return ref_dist(a.x32 + row * a.dim, cb + j * a.dim, a.dim);
}
__device__ __forceinline__ float rin_of(const KernelArgs& a, long long row) { return a.rin ? a.rin[row] : 0.f; }

// A pass kernel has nothing to do once the design is done or when the fused
// small-codebook pass (pass_small_kernel) already ran this pass.
__device__ __forceinline__ bool pass_off(const DevState* st) { return st->done || st->skip; }

// Programmatic dependent launch: pass kernels are launched with
// programmaticStreamSerialization (launch_k), so a kernel's grid is set up
// while its predecessor drains; each begins with pdl_wait(), which returns
// once the predecessor has completed and its writes are visible (a no-op for
// a kernel launched without the attribute).  VQB_PDL=0 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Extra certified band for float64 rows rounded to float32 (rn = rin[row]):
// the reference compares d_j = ||x - c_j||^2 while the candidate pass sees
// x^ = fl32(x); d_j - d_1 moves by 2 (x - x^).(c_1 - c_j), at most
// 2 rn (sqrt d_1 + sqrt d_j).  With B >= every sqrt d inside the band (from
// the best value m1 + q and the FP band 3E) the extra term 4 rn B + 2 rn^2
// keeps "certified" and "the reference's winner lies inside the band" true.
__host__ __device__ __forceinline__ float input_band(float rn, float d1, float e3) {
  if (!(rn > 0.f)) return 0.f;
  const float B = (sqrtf(fmaxf(d1 + e3, 0.f)) + 4.0f * rn) * 1.02f;
  return 4.0f * rn * B + 2.0f * rn * rn;
}

// kernel launchers (kernels.cu); all asynchronous on `stream`
cudaError_t launch_prep_codebook(const KernelArgs& a, cudaStream_t s);
cudaError_t launch_assign(const KernelArgs& a, bool fast, int sms, cudaStream_t s);
cudaError_t launch_rerank(const KernelArgs& a, int sms, cudaStream_t s);
bool shortlist_enabled();
cudaError_t launch_epilogue(const KernelArgs& a, bool want_dists, bool want_sums, bool zero_cells,
                            int sms, cudaStream_t s);
// reference-order FP64 cell sums (update_rows' ascending-index order): stable
// counting sort of the rows by cell, then one sequential FP64 chain per
// (cell, dimension); zero_cells: every row in cell 0 (the initial centroid)
cudaError_t launch_ordered_update(const KernelArgs& a, bool zero_cells, int sms, cudaStream_t s);
int ordered_blocks(long long n);
cudaError_t launch_finalize(const KernelArgs& a, bool stage, cudaStream_t s);
// the fused single-kernel pass for small codebooks (training loop, one device)
cudaError_t launch_pass_small(const KernelArgs& a, int sms, cudaStream_t s);
cudaError_t launch_init_centroid(const KernelArgs& a, bool stage, cudaStream_t s);
cudaError_t launch_clear(const KernelArgs& a, cudaStream_t s);
cudaError_t launch_maxabs(const float* x32, const double* x64, long long count,
                          unsigned long long* out_bits, int sms, cudaStream_t s);
// per-column max |x| (FP64 bit patterns, NaN bits for a non-finite value) and
// lowest set bit exponent (INT_MAX for a column of zeros) of rows x[rows][dim]
cudaError_t launch_colstats(const float* x32, const double* x64, long long rows, int dim,
                            unsigned long long* cmax, int* clow, int sms, cudaStream_t s);
cudaError_t launch_colstats_reset(unsigned long long* cmax, int* clow, int dim, cudaStream_t s);
// per-column shifts (cshift) + lo_shift / sums_exact / ref_exact / nonfinite
// from column stats, on the device (the host-buffer Lloyd step)
cudaError_t launch_set_shift(DevState* st, const unsigned long long* cmax, const int* clow, int dim,
                             long long n_global, int* cshift, unsigned long long* maxabs_bits, cudaStream_t s);
cudaError_t launch_widen_idx(const int* idx, long long* out, long long n, int sms, cudaStream_t s);
cudaError_t launch_sum_inorder(const double* v, long long n, double* out, cudaStream_t s);
cudaError_t launch_reset(DevState* st, int mode, int size, int metric, int ordered, int keep_cur,
                         cudaStream_t s);
cudaError_t launch_cells_to_idx(const long long* cells, int* idx, long long n, int sms, cudaStream_t s);
cudaError_t launch_f64_to_f32_exact(const double* x64, float* x32, long long count, int* inexact,
                                    int sms, cudaStream_t s);
cudaError_t launch_column_sums_ordered(const double* x64, const float* x32, long long m, int dim,
                                       double* out, cudaStream_t s);
cudaError_t launch_pair_distance(const double* a, const double* b, int dim, int metric, double* out,
                                 cudaStream_t s);
bool fast_dim_supported(int dim);
// candidate width of a row length: 16 / 32 / 64, or 0 (no fast path, L > 64)
inline int candidate_dim(int dim) { return dim <= 16 ? 16 : (dim <= 32 ? 32 : (dim <= 64 ? 64 : 0)); }
// fl32 + zero-padded candidate copy of rows (x64 or x32, [n][dim] -> [n][cdim])
// and, for float64 rows, the per-row rounding bound rin
cudaError_t launch_candidate_rows(const float* x32, const double* x64, long long n, int dim, int cdim,
                                  float* xc, float* rin, int sms, cudaStream_t s);

// Gaussian-mixture rows on the device (gmm.cu): means [comps][dim] f32,
// sigmas [comps] f32, cw [comps] cumulative weights (nullable: uniform)
cudaError_t launch_gmm_rows(const float* means, const float* sigmas, const double* cw, long long comps,
                            long long rows, int dim, long long row0, unsigned long long seed, float* out, int sms,
                            cudaStream_t s);

// block vectoriser / decode / reconstruction distortion (imaging.cu)
cudaError_t launch_pixels_to_blocks_f32(const unsigned char* px, long long images, long long H, long long W,
                                        int block, float* out, cudaStream_t s);
cudaError_t launch_pixels_to_blocks_f64(const unsigned char* px, long long images, long long H, long long W,
                                        int block, double* out, cudaStream_t s);
// vecs[count][block^2] (or, with vecs == nullptr, codebook rows cb[idx[v]]) -> pixels
cudaError_t launch_blocks_to_pixels(const double* vecs, const unsigned* idx, const double* cb, long long images,
                                    long long H, long long W, int block, unsigned char* out, cudaStream_t s);
// decode fused with the raster; cbq = K * block^2 bytes of scratch
cudaError_t launch_decode_pixels(const unsigned* idx, const double* cb, long long K, long long images,
                                 long long H, long long W, int block, unsigned char* cbq, unsigned char* out,
                                 cudaStream_t s);
cudaError_t launch_decode(const unsigned* idx, long long n, int L, const double* cb, long long K, double* out,
                          int* bad, cudaStream_t s);
cudaError_t launch_split_rows(const double* cb, long long size, int dim, double delta, double* out,
                              cudaStream_t s);
cudaError_t launch_index_check(const unsigned* idx, long long n, long long K, int* bad, cudaStream_t s);
cudaError_t launch_pair_rows(const double* a, const double* b, long long n, int dim, int metric, double* d,
                             cudaStream_t s);
cudaError_t launch_distortion_sum(const double* d, long long n, bool inorder, double* tiles, double* out,
                                  cudaStream_t s);

// tensor-core candidate pass (assign_tc.cu)
constexpr int kTcChunk = 256;  // codewords per MMA N
constexpr int kTcRows = 128;   // rows per tile (MMA M)
constexpr int kTcShort = 8;    // shortlist candidates per row before the full FP64 scan
// queued rows x codebook size below which the FP32 shortlist (warp per row)
// rescans instead of the TC shortlist pass: a short queue at a small codebook
// does not pay the TC pass's per-CTA set-up (cfg2 K=64: 19.5 -> 13.4 us);
// either is valid for TC-flagged rows (the FP32 error is below the TC band's)
#ifndef VQB_TC_SL_WORK
#define VQB_TC_SL_WORK (1LL << 19)
#endif
constexpr long long kTcShortlistWork = VQB_TC_SL_WORK;
__host__ __device__ inline long long tc_chunk_elems(int dim) { return (long long)kTcChunk * (2 * dim + 16); }
int tc_max_size(int dim);      // largest codebook whose operand image fits in smem
// does assign_tc (rather than assign_fast) run the candidate pass at size K?
__host__ __device__ __forceinline__ bool tc_handles(const DevState* st, int K) {
  // one chunk of N = K columns (K = 64, 128) or whole 256-column chunks
  return st->tc_on && !st->tc_bad && K >= st->tc_kmin && K <= st->tc_kmax &&
         (K % kTcChunk == 0 || K == 64 || K == 128);
}
cudaError_t launch_assign_tc(const KernelArgs& a, int sms, cudaStream_t s);
cudaError_t launch_shortlist_tc(const KernelArgs& a, int sms, cudaStream_t s);
cudaError_t launch_tc_probe(const KernelArgs& a, float* dump, cudaStream_t s);
// the rows' operand image for the current tc_ey (rows [0, n) of x32)
cudaError_t launch_build_row_image(const float* x32, const float* mu, long long n, int dim, int ey,
                                   unsigned short* aimg, float* aq, int sms, cudaStream_t s);
__host__ __device__ inline long long tc_row_image_elems(long long n, int dim) {
  return (n + kTcRows - 1) / kTcRows * (2LL * kTcRows * dim);
}

// element offset of (row, col) in a K-major, no-swizzle UMMA operand tile with
// kt columns: 8-row x 16-byte core matrices, K-adjacent core matrices 128 B
// apart (LBO), 8-row groups kt*16 B apart (SBO)
__host__ __device__ __forceinline__ long long tc_off(int row, int col, int kt) {
  return (long long)(row >> 3) * (kt * 8) + (col >> 3) * 64 + (row & 7) * 8 + (col & 7);
}

// fp16 hi/lo image of staged codevector k (w = -2 c~ in FP32, nrm = ||c~||^2
// in FP64): chunk k/256 = [wh 256 x L | wl 256 x L | wn 256 x 16], where
// wh + wl = w * 2^ew and 2^kn (nh + nl) = nrm * 2^(ey + ew).  Values fp16
// cannot hold set tc_bad, which sends the pass to the FP32 kernel.
__device__ __forceinline__ void stage_tc_row(const KernelArgs& a, long long k, const float* w, double nrm) {
  if (!a.tcb) return;
  DevState* st = a.st;
  const int L = a.cdim;
  unsigned short* img = a.tcb + (k / kTcChunk) * tc_chunk_elems(L);
  const int r = (int)(k % kTcChunk);
  unsigned short* wh = img;
  unsigned short* wl = img + (long long)kTcChunk * L;
  unsigned short* wn = img + 2LL * kTcChunk * L;
  const float sw = ldexpf(1.0f, st->tc_ew);
  bool bad = false;
  for (int l = 0; l < L; ++l) {
    const float v = w[l] * sw;
    const __half h = __float2half_rn(v);
    const __half lo = __float2half_rn(v - __half2float(h));
    bad |= !(fabsf(v) <= 60000.0f);
    wh[tc_off(r, l, L)] = __half_as_ushort(h);
    wl[tc_off(r, l, L)] = __half_as_ushort(lo);
  }
  const double nv = ldexp(nrm, st->tc_ey + st->tc_ew - st->tc_kn);
  const __half nh = __double2half(nv);
  const __half nl = __double2half(nv - (double)__half2float(nh));
  bad |= !(fabs(nv) <= 60000.0);
  for (int c = 0; c < 16; ++c)
    wn[tc_off(r, c, 16)] = c == 0 ? __half_as_ushort(nh) : (c == 1 ? __half_as_ushort(nl) : 0);
  if (bad) st->tc_bad = 1;
}

}  // namespace vqb
