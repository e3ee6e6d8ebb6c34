// C ABI + native LBG driver loop (see include/vqb200.h for the contract and
// the reference interfaces each entry point replaces).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vqb200.h"
#include "transfer.h"
#include "vqb200_internal.h"

using namespace vqb;

// the part of DevState the host writes / reads back (everything before the
// history buffer fields)
static constexpr size_t kStateHeader = offsetof(DevState, hist_cap);

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(VQB_INTERNAL, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, \
                  __LINE__, cudaGetErrorString(e_));                                      \
  } while (0)

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
}


}  // namespace

struct vqb_session {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // H2D pieces (transfer.cpp), overlapped with kernels
  bool own_stream = false;
  long long n = 0, dim = 0, row_offset = 0, n_global = 0;
  float* x32 = nullptr;
  double* x64 = nullptr;
  // candidate rows of the FP32 / TC passes (KernelArgs::xc): fl32 + zero pad
  // to cdim (== x32 when the rows are float32 of a candidate width)
  float* xc_own = nullptr;
  float* rin = nullptr;  // float64 rows: per-row rounding bound
  int cdim = 0;          // 16 / 32 / 64, or 0: no candidate pass
  float* mu = nullptr;
  std::vector<float> mu_host;  // host copy of the centring vector
  double maxabs = -1.0;
  // per-column stats of this shard's rows (colstats): max |x| and the lowest
  // set bit exponent -- the two-word fixed-point plan of the cell sums
  std::vector<double> colmax;
  std::vector<int> collow;
  std::vector<int> cshift_host;
  unsigned long long* cmax = nullptr;  // device copies (host-buffer paths recompute them per call)
  int* clow = nullptr;
  int* cshift = nullptr;               // per-column shifts of the current run
  bool sums_exact = true, ref_exact = true;
  // history: a device ring the finalize kernel writes, drained by the host
  // after every batch of passes (so a run may record any number of passes)
  HistRec* hist = nullptr;
  int hist_cap = 0;
  long long drained = 0;                       // records copied to hist_raw so far
  std::vector<HistRec> hist_raw;
  std::vector<vqb_level_iteration> hist_host;  // the last run's history (vqb_step_history)
  // reference-order cell sums (ordered.cu), allocated on first use
  int* operm = nullptr;
  int* obase = nullptr;
  int* oscan = nullptr;
  int oblocks = 0;
  long long obase_k = 0;
  // one caller at a time: ctypes releases the GIL, and every call below uses
  // the session's buffers, state and pinned arena
  std::recursive_mutex lock_mu;
  unsigned short* tcb = nullptr;  // fp16 operand image of the codebook (assign_tc)
  // fp16 operand image of the resident rows (assign_tc reads it with bulk
  // copies instead of converting every pass); built for scale 2^aimg_ey
  bool rows_resident = false;  // x32 holds the session's rows for its lifetime (vqb_open)
  unsigned short* aimg = nullptr;
  float* aq = nullptr;
  int aimg_ey = INT_MIN;
  // run buffers
  long long kmax = 0;
  double* cb[2] = {nullptr, nullptr};
  float* w = nullptr;
  float* nrm = nullptr;
  int* idx = nullptr;
  int* flags = nullptr;
  float* flag_thr = nullptr;
  int* flags2 = nullptr;
  double* dists = nullptr;
  long long* ex = nullptr;
  long long* partials = nullptr;
  double* ord = nullptr;
  long long ntiles_global = 0;
  DevState* st = nullptr;
  DevState* st_host = nullptr;  // pinned
  int* done_host = nullptr;     // pinned
  double* scratch = nullptr;    // small device scratch
  bool fast = false;
  bool ordered = false;
  bool fused_ok = false;  // vqb_train on one device: the fused small-codebook pass leads every pass
  // incremental cell sums of the training loop (kernels.cu moved_scan_kernel):
  // previous cells, moved list, running local sums; allocated by the first design
  int* idx_prev = nullptr;
  int* mv = nullptr;
  long long* acc = nullptr;
  bool delta_on = false;
  double delta_frac = 0.3;
  bool pending_init = false;
  long long lloyd_size = 0;  // vqb_lloyd_begin
  cudaEvent_t ev_batch[2] = {nullptr, nullptr};
  // pinned host arena for small per-call transfers (codebooks, centre) so
  // they never take the synchronous pageable-copy path; reset per call
  char* pin = nullptr;
  size_t pin_cap = 0, pin_off = 0;
  std::vector<cudaEvent_t> piece_ev;  // H2D piece completions (host-buffer paths)
  // captured batch of training passes (vqb_train); rebuilt when buffers or the
  // pass shape (fast / ordered) change
  cudaGraphExec_t graph = nullptr;
  long long graph_kmax = -1;
  int graph_key = -1;
  int batch_graph(int batch);
  void drop_graph() {
    if (graph) cudaGraphExecDestroy(graph);
    graph = nullptr;
    graph_kmax = -1;
    graph_key = -1;
  }

  char* pin_alloc(size_t bytes) {
    bytes = (bytes + 255) / 256 * 256;
    if (pin_off + bytes > pin_cap) return nullptr;
    char* p = pin + pin_off;
    pin_off += bytes;
    return p;
  }
  int pin_reserve(size_t bytes) {
    if (bytes <= pin_cap) return VQB_OK;
    if (stream) cudaStreamSynchronize(stream);
    if (pin) cudaFreeHost(pin);
    pin = nullptr;
    pin_cap = 0;
    CK(cudaMallocHost(reinterpret_cast<void**>(&pin), bytes));
    pin_cap = bytes;
    return VQB_OK;
  }

  KernelArgs args() const {
    KernelArgs a{};
    a.x32 = x32;
    a.x64 = x64;
    a.cdim = cdim ? cdim : (int)dim;
    a.xc = xc_own ? xc_own : (cdim == dim ? x32 : nullptr);
    a.rin = rin;
    a.n = n;
    a.n_global = n_global;
    a.r0 = 0;
    a.r1 = n;
    a.dim = (int)dim;
    a.tile0 = row_offset / kTdTile;
    a.mu = mu;
    a.cshift = cshift;
    a.cb[0] = cb[0];
    a.cb[1] = cb[1];
    a.w = w;
    a.tcb = tcb;
    a.aimg = aimg_ey != INT_MIN ? aimg : nullptr;
    a.aq = aimg_ey != INT_MIN ? aq : nullptr;
    a.nrm = nrm;
    a.kmax = kmax;
    a.idx = idx;
    a.flags = flags;
    a.flag_thr = flag_thr;
    a.flags2 = flags2;
    a.dists = dists;
    a.ex.base = ex;
    a.ex.kmax = kmax;
    a.ex.dim = dim;
    a.ex.ntiles = ntiles_global;
    a.partials = partials;
    a.ord = ord;
    a.operm = operm;
    a.obase = obase;
    a.oscan = oscan;
    a.oblocks = oblocks;
    a.idx_prev = delta_on ? idx_prev : nullptr;
    a.mv = delta_on ? mv : nullptr;
    a.mv_cap = n + 32;
    a.acc = delta_on ? acc : nullptr;
    a.delta_max = (long long)((double)n * delta_frac);
    static const int small = [] {
      const char* e = getenv("VQB_SMALL");
      return e ? atoi(e) : 1;
    }();
    a.small_on = small;
    static const int diff = [] {
      const char* e = getenv("VQB_DIFF");
      return e ? atoi(e) : 1;
    }();
    a.diff_on = diff;
    a.st = st;
    return a;
  }

  int ensure(long long k) {
    if (k <= kmax && cb[0]) return VQB_OK;
    drop_graph();
    cudaFree(cb[0]);
    cudaFree(cb[1]);
    cudaFree(w);
    cudaFree(nrm);
    cudaFree(ex);
    cudaFree(partials);
    cudaFree(ord);
    cudaFree(tcb);
    cudaFree(acc);
    acc = nullptr;
    ord = nullptr;
    tcb = nullptr;
    cb[0] = cb[1] = nullptr;
    w = nrm = nullptr;
    ex = nullptr;
    partials = nullptr;
    kmax = k;
    const long long kpad = (k + 3) / 4 * 4;
    CK(dalloc(&cb[0], (size_t)(k * dim)));
    CK(dalloc(&cb[1], (size_t)(k * dim)));
    const long long wd = cdim > dim ? cdim : dim;
    CK(dalloc(&w, (size_t)(kpad * wd + 64)));
    CK(dalloc(&nrm, (size_t)(kpad + 64)));
    CK(dalloc(&ex, (size_t)(2 * k * dim + k + ntiles_global)));  // Exchange::words()
    CK(dalloc(&partials, (size_t)sms * (size_t)(k * dim + k)));
    CK(dalloc(&ord, (size_t)(k * dim)));
    if (fast_dim_supported(cdim))
      CK(dalloc(&tcb, (size_t)(((k + kTcChunk - 1) / kTcChunk) * tc_chunk_elems(cdim))));
    CK(cudaMemsetAsync(ex, 0, sizeof(long long) * (2 * k * dim + k + ntiles_global), stream));
    return VQB_OK;
  }

  ~vqb_session() {
    if (device >= 0) cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    cudaFree(x32);
    cudaFree(x64);
    cudaFree(xc_own);
    cudaFree(rin);
    cudaFree(mu);
    cudaFree(cb[0]);
    cudaFree(cb[1]);
    cudaFree(w);
    cudaFree(nrm);
    cudaFree(idx);
    cudaFree(flags);
    cudaFree(flag_thr);
    cudaFree(flags2);
    cudaFree(dists);
    cudaFree(ex);
    cudaFree(partials);
    cudaFree(ord);
    cudaFree(tcb);
    cudaFree(aimg);
    cudaFree(aq);
    cudaFree(cmax);
    cudaFree(clow);
    cudaFree(cshift);
    cudaFree(hist);
    cudaFree(operm);
    cudaFree(obase);
    cudaFree(oscan);
    cudaFree(idx_prev);
    cudaFree(mv);
    cudaFree(acc);
    cudaFree(st);
    cudaFree(scratch);
    if (st_host) cudaFreeHost(st_host);
    if (done_host) cudaFreeHost(done_host);
    for (auto& e : ev_batch)
      if (e) cudaEventDestroy(e);
    for (auto& e : piece_ev) cudaEventDestroy(e);
    if (pin) cudaFreeHost(pin);
    drop_graph();
    if (own_stream && stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
  }

  int make_streams() {
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    own_stream = true;
    return VQB_OK;
  }

  // device buffers every session needs besides the rows
  int alloc_common() {
    CK(dalloc(&idx, (size_t)n + 32));
    CK(dalloc(&flags, (size_t)n + 32));
    CK(dalloc(&flag_thr, (size_t)n + 32));
    CK(dalloc(&flags2, (size_t)n + 32));
    CK(dalloc(&dists, (size_t)n + 32));
    CK(dalloc(&st, 1));
    CK(cudaMemset(st, 0, sizeof(DevState)));  // every field starts defined (skip, barriers, ...)
    CK(dalloc(&mu, (size_t)dim + 68));  // zero-padded up to the candidate width
    CK(cudaMemset(mu, 0, sizeof(float) * (dim + 68)));
    CK(dalloc(&cmax, (size_t)dim));
    CK(dalloc(&clow, (size_t)dim));
    CK(dalloc(&cshift, (size_t)dim));
    CK(cudaMemset(cshift, 0, sizeof(int) * dim));
    CK(cudaMallocHost(reinterpret_cast<void**>(&st_host), sizeof(DevState)));
    std::memset(st_host, 0, sizeof(DevState));
    CK(cudaMallocHost(reinterpret_cast<void**>(&done_host), 4 * sizeof(int)));
    return alloc_hist();
  }

  // the history ring (VQB_HIST_RING overrides its size, for tests); the
  // device state points at it
  int alloc_hist() {
    static const int ring = [] {
      const char* e = getenv("VQB_HIST_RING");
      const int v = e ? atoi(e) : kHistRing;
      return v >= 16 ? v : kHistRing;
    }();
    CK(dalloc(&hist, (size_t)ring));
    hist_cap = ring;
    // hist_cap / hist close DevState: the header copies (kStateHeader bytes)
    // never overwrite them
    CK(cudaMemcpy(reinterpret_cast<char*>(st) + offsetof(DevState, hist_cap), &hist_cap, sizeof(int),
                  cudaMemcpyHostToDevice));
    CK(cudaMemcpy(reinterpret_cast<char*>(st) + offsetof(DevState, hist), &hist, sizeof(HistRec*),
                  cudaMemcpyHostToDevice));
    return VQB_OK;
  }

  // copy the ring's records [drained, upto) to the host (they were written by
  // passes that have completed; the copy runs on the copy stream, so it does
  // not queue behind the batch the device is executing now)
  int drain_hist(long long upto) {
    if (upto <= drained) return VQB_OK;
    if (upto - drained > hist_cap)
      return fail(VQB_INTERNAL, "history ring overrun (%lld records pending, ring %d)", upto - drained, hist_cap);
    const size_t old = hist_raw.size();
    hist_raw.resize((size_t)upto);
    long long i = drained;
    while (i < upto) {
      const long long slot = i % hist_cap;
      const long long run = std::min<long long>(upto - i, hist_cap - slot);
      CK(cudaMemcpyAsync(hist_raw.data() + old + (i - drained), hist + slot, sizeof(HistRec) * run,
                         cudaMemcpyDeviceToHost, copy_stream));
      i += run;
    }
    CK(cudaStreamSynchronize(copy_stream));
    drained = upto;
    return VQB_OK;
  }

  // buffers of the incremental cell sums (VQB_DELTA=0 turns them off;
  // VQB_DELTA_FRAC: the moved fraction up to which a pass updates the running
  // sums instead of summing every row)
  int ensure_delta() {
    const char* e = getenv("VQB_DELTA");
    delta_on = !(e && strcmp(e, "0") == 0);
    if (!delta_on) return VQB_OK;
    const char* f = getenv("VQB_DELTA_FRAC");
    const double v = f ? atof(f) : 0.3;
    delta_frac = v >= 0.0 && v <= 1.0 ? v : 0.3;
    if (!idx_prev) {
      drop_graph();
      CK(dalloc(&idx_prev, (size_t)n + 32));
      CK(cudaMemsetAsync(idx_prev, 0xff, sizeof(int) * (n + 32), stream));
    }
    if (!mv) CK(dalloc(&mv, (size_t)(3 * (n + 32))));
    if (!acc) {
      drop_graph();
      CK(dalloc(&acc, (size_t)(2 * kmax * dim + kmax)));
      CK(cudaMemsetAsync(acc, 0, sizeof(long long) * (2 * kmax * dim + kmax), stream));
    }
    return VQB_OK;
  }

  // buffers of the reference-order path for codebooks up to k
  int ensure_ordered(long long k) {
    const int B = ordered_blocks(n);
    if (operm && obase_k >= k && oblocks == B) return VQB_OK;
    drop_graph();
    cudaFree(operm);
    cudaFree(obase);
    cudaFree(oscan);
    operm = obase = oscan = nullptr;
    oblocks = B;
    obase_k = k;
    CK(dalloc(&operm, (size_t)n + 32));
    CK(dalloc(&obase, (size_t)(k * B)));
    CK(dalloc(&oscan, (size_t)((k * B + 4095) / 4096 + 256)));
    return VQB_OK;
  }

  // Two-word fixed-point plan of the cell sums from column stats (this
  // shard's, or the global ones every rank agreed on): per-column shifts to
  // the device, lo_shift and the exactness flags into the host state `h`.
  int plan_fixed(DevState* h, const double* gmax = nullptr, const int* glow = nullptr) {
    cshift_host.assign((size_t)dim, 0);
    bool ex = true, rex = true;
    const bool have = (long long)colmax.size() == dim;  // host-buffer sessions plan on the device
    for (long long l = 0; l < dim; ++l) {
      const double m = gmax ? gmax[l] : (have ? colmax[(size_t)l] : 0.0);
      const int lw = glow ? glow[l] : (have ? collow[(size_t)l] : 0x7fffffff);
      const FixedCol f = fixed_plan(n_global, m, lw);
      cshift_host[(size_t)l] = f.s;
      ex = ex && f.exact;
      rex = rex && f.ref_exact;
    }
    sums_exact = ex;
    ref_exact = rex;
    h->lo_shift = fixed_lo_shift(n_global);
    h->sums_exact = ex ? 1 : 0;
    h->ref_exact = rex ? 1 : 0;
    char* p = pin_alloc(sizeof(int) * dim);
    if (p) std::memcpy(p, cshift_host.data(), sizeof(int) * dim);
    CK(cudaMemcpyAsync(cshift, p ? static_cast<const void*>(p) : cshift_host.data(), sizeof(int) * dim,
                       cudaMemcpyHostToDevice, stream));
    return VQB_OK;
  }
};

extern "C" {

const char* vqb_last_error(void) { return g_err.c_str(); }
int vqb_version(void) { return 1; }

int vqb_device_count(int* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
    return fail(VQB_INTERNAL, "no CUDA device: %s", cudaGetErrorString(e));
  }
  *count = c;
  return VQB_OK;
}

}  // extern "C"

// Validation + session shell shared by vqb_open and vqb_open_pixels.
static int new_session(int64_t rows, int64_t dim, int64_t row_offset, int64_t n_global, int device,
                       std::unique_ptr<vqb_session>& s) {
  if (rows < 1 || dim < 1)
    return fail(VQB_USAGE, "training set must be at least 1x1, got %lldx%lld", (long long)rows,
                (long long)dim);
  if (n_global < rows + row_offset || row_offset < 0)
    return fail(VQB_USAGE, "shard [%lld, %lld) outside %lld global rows", (long long)row_offset,
                (long long)(row_offset + rows), (long long)n_global);
  if (row_offset % kTdTile != 0)
    return fail(VQB_USAGE, "shard offset %lld must be a multiple of %d rows", (long long)row_offset,
                kTdTile);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(VQB_INTERNAL, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  CK(cudaSetDevice(device));
  s.reset(new vqb_session());
  s->device = device;
  CK(cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, device));
  if (int rc = s->make_streams()) return rc;
  s->n = rows;
  s->dim = dim;
  s->row_offset = row_offset;
  s->n_global = n_global;
  s->ntiles_global = (n_global + kTdTile - 1) / kTdTile;
  CK(dalloc(&s->scratch, 64));
  return VQB_OK;
}

static int finish_open(std::unique_ptr<vqb_session>& s, vqb_session** out);

extern "C" {

int vqb_open(const float* x32, const double* x64, int64_t rows, int64_t dim, int64_t row_offset,
             int64_t n_global, int device, vqb_session** out) {
  *out = nullptr;
  if ((x32 == nullptr) == (x64 == nullptr))
    return fail(VQB_USAGE, "exactly one of x32 / x64 must be given");
  std::unique_ptr<vqb_session> s;
  if (int rc = new_session(rows, dim, row_offset, n_global, device, s)) return rc;
  const size_t count = (size_t)rows * dim;
  if (x32) {
    CK(dalloc(&s->x32, count + 16));
    CK(upload(s->x32, x32, count * sizeof(float), 16u << 20, s->copy_stream, s->stream));
  } else {
    CK(dalloc(&s->x64, count + 8));
    CK(upload(s->x64, x64, count * sizeof(double), 16u << 20, s->copy_stream, s->stream));
    // float64 rows that are exactly float32 take the FP32 candidate path
    float* tmp = nullptr;
    CK(dalloc(&tmp, count + 16));
    int* flag = reinterpret_cast<int*>(s->scratch);
    CK(cudaMemsetAsync(flag, 0, sizeof(int), s->stream));
    CK(launch_f64_to_f32_exact(s->x64, tmp, (long long)count, flag, s->sms, s->stream));
    int inexact = 1;
    CK(cudaMemcpyAsync(&inexact, flag, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    if (!inexact) {
      cudaFree(s->x64);
      s->x64 = nullptr;
      s->x32 = tmp;
    } else {
      cudaFree(tmp);
    }
  }
  return finish_open(s, out);
}

int vqb_open_pixels(const uint8_t* pixels, int64_t images, int64_t height, int64_t width, int64_t block,
                    int device, vqb_session** out) {
  *out = nullptr;
  if (images < 1 || height < 1 || width < 1)
    return fail(VQB_USAGE, "image must be at least 1x1, got %lldx%lld", (long long)width, (long long)height);
  if (block < 1) return fail(VQB_USAGE, "block side must be >= 1, got %lld", (long long)block);
  if (block > 4096) return fail(VQB_USAGE, "block side %lld too large", (long long)block);
  const long long per_img = ((height + block - 1) / block) * ((width + block - 1) / block);
  const long long rows = per_img * images;
  std::unique_ptr<vqb_session> s;
  if (int rc = new_session(rows, block * block, 0, rows, device, s)) return rc;
  const size_t npx = (size_t)(images * height * width);
  unsigned char* dpx = nullptr;
  CK(dalloc(&dpx, npx));
  std::unique_ptr<unsigned char, decltype(&cudaFree)> g(dpx, &cudaFree);
  CK(dalloc(&s->x32, (size_t)rows * block * block + 16));
  CK(upload(dpx, pixels, npx, 16u << 20, s->copy_stream, s->stream));
  CK(launch_pixels_to_blocks_f32(dpx, images, height, width, (int)block, s->x32, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return finish_open(s, out);
}

int vqb_open_gmm(const float* means, const float* sigmas, const double* cum_weights, int64_t components,
                 int64_t rows, int64_t dim, int64_t row_offset, int64_t n_global, uint64_t seed, int device,
                 vqb_session** out) {
  *out = nullptr;
  if (!means || !sigmas) return fail(VQB_USAGE, "means and sigmas are required");
  if (components < 1) return fail(VQB_USAGE, "mixture needs at least one component, got %lld", (long long)components);
  for (int64_t i = 0; i < components * dim; ++i)
    if (!std::isfinite(means[i])) return fail(VQB_USAGE, "mean %lld is not finite", (long long)i);
  for (int64_t i = 0; i < components; ++i)
    if (!std::isfinite(sigmas[i]) || sigmas[i] < 0.f)
      return fail(VQB_USAGE, "sigma %lld must be finite and >= 0", (long long)i);
  if (cum_weights) {
    for (int64_t i = 0; i < components; ++i)
      if (!(cum_weights[i] >= (i ? cum_weights[i - 1] : 0.0)) || cum_weights[i] > 1.0)
        return fail(VQB_USAGE, "cumulative weights must be nondecreasing in [0, 1] (entry %lld)", (long long)i);
    if (cum_weights[components - 1] != 1.0) return fail(VQB_USAGE, "cumulative weights must end at 1");
  }
  std::unique_ptr<vqb_session> s;
  if (int rc = new_session(rows, dim, row_offset, n_global, device, s)) return rc;
  float *dm = nullptr, *dsg = nullptr;
  double* dcw = nullptr;
  CK(dalloc(&dm, (size_t)(components * dim)));
  std::unique_ptr<float, decltype(&cudaFree)> g0(dm, &cudaFree);
  CK(dalloc(&dsg, (size_t)components));
  std::unique_ptr<float, decltype(&cudaFree)> g1(dsg, &cudaFree);
  if (cum_weights) CK(dalloc(&dcw, (size_t)components));
  std::unique_ptr<double, decltype(&cudaFree)> g2(dcw, &cudaFree);
  CK(cudaMemcpyAsync(dm, means, sizeof(float) * components * dim, cudaMemcpyHostToDevice, s->stream));
  CK(cudaMemcpyAsync(dsg, sigmas, sizeof(float) * components, cudaMemcpyHostToDevice, s->stream));
  if (dcw) CK(cudaMemcpyAsync(dcw, cum_weights, sizeof(double) * components, cudaMemcpyHostToDevice, s->stream));
  CK(dalloc(&s->x32, (size_t)rows * dim + 16));
  CK(launch_gmm_rows(dm, dsg, dcw, components, rows, (int)dim, row_offset, (unsigned long long)seed, s->x32,
                     s->sms, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return finish_open(s, out);
}

}  // extern "C"

static int finish_open(std::unique_ptr<vqb_session>& s, vqb_session** out) {
  const long long rows = s->n, dim = s->dim;
  if (int rc = s->alloc_common()) return rc;
  // per-column max |x| and lowest set bit (fixed-point plan of the cell
  // sums; max |x| also decides fast-path eligibility)
  CK(launch_colstats_reset(s->cmax, s->clow, (int)dim, s->stream));
  CK(launch_colstats(s->x32, s->x64, rows, (int)dim, s->cmax, s->clow, s->sms, s->stream));
  std::vector<unsigned long long> cm((size_t)dim);
  s->collow.assign((size_t)dim, 0);
  CK(cudaMemcpyAsync(cm.data(), s->cmax, sizeof(unsigned long long) * dim, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(s->collow.data(), s->clow, sizeof(int) * dim, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaEventCreateWithFlags(&s->ev_batch[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s->ev_batch[1], cudaEventDisableTiming));
  CK(cudaStreamSynchronize(s->stream));
  s->colmax.assign((size_t)dim, 0.0);
  s->maxabs = 0.0;
  for (long long l = 0; l < dim; ++l) {
    double v;
    std::memcpy(&v, &cm[(size_t)l], sizeof(double));
    if (!(v <= 1.7976931348623157e308)) v = INFINITY;
    s->colmax[(size_t)l] = v;
    s->maxabs = std::max(s->maxabs, v);
  }
  {
    // exactness of this shard's own fixed-point plan (the summation mode of
    // single-device calls; a sharded run re-plans from the global stats)
    bool ex = true, rex = true;
    for (long long l = 0; l < dim; ++l) {
      const FixedCol f = fixed_plan(s->n_global, s->colmax[(size_t)l], s->collow[(size_t)l]);
      ex = ex && f.exact;
      rex = rex && f.ref_exact;
    }
    s->sums_exact = ex;
    s->ref_exact = rex;
  }
  // centring vector: the shard's first row mean is as good as any; use a
  // cheap, deterministic one -- the midpoint of [-maxabs, maxabs] is 0, so
  // centre at the column means of up to 4096 leading rows (FP32, host-free:
  // computed from the device copy).
  {
    std::vector<float> h((size_t)std::min<long long>(rows, 4096) * dim);
    std::vector<double> h64;
    const long long m = std::min<long long>(rows, 4096);
    if (s->x32) {
      CK(cudaMemcpy(h.data(), s->x32, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
    } else {
      h64.resize(h.size());
      CK(cudaMemcpy(h64.data(), s->x64, h64.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < h.size(); ++i) h[i] = (float)h64[i];
    }
    std::vector<float> mu((size_t)dim, 0.f);
    for (long long l = 0; l < dim; ++l) {
      double acc = 0;
      for (long long j = 0; j < m; ++j) acc += h[(size_t)j * dim + l];
      mu[(size_t)l] = std::isfinite(acc) ? (float)(acc / (double)m) : 0.f;
    }
    CK(cudaMemcpy(s->mu, mu.data(), dim * sizeof(float), cudaMemcpyHostToDevice));
    s->mu_host = mu;
  }
  // candidate rows: the FP32 / tensor-core pass runs for every L <= 64 (rows
  // zero-padded to 16 / 32 / 64) and for float64 rows (rounded to float32,
  // the rounding bounded per row and added to the certified band)
  s->cdim = candidate_dim((int)dim);
  if (s->cdim && (s->x64 || s->cdim != dim)) {
    CK(dalloc(&s->xc_own, (size_t)rows * s->cdim + 16));
    if (s->x64) CK(dalloc(&s->rin, (size_t)rows + 16));
    CK(launch_candidate_rows(s->x32, s->x64, rows, (int)dim, s->cdim, s->xc_own, s->rin, s->sms, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  }
  s->fast = s->cdim != 0 && s->maxabs < 1099511627776.0;
  s->rows_resident = true;
  *out = s.release();
  return VQB_OK;
}

extern "C" {

int vqb_rows_f32(vqb_session* s, float* out) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  if (!s->x32) return fail(VQB_USAGE, "the session holds float64 rows");
  CK(cudaSetDevice(s->device));
  CK(download(out, s->x32, sizeof(float) * (size_t)(s->n * s->dim), s->stream));
  return VQB_OK;
}

int vqb_close(vqb_session* s) {
  delete s;
  return VQB_OK;
}

int vqb_set_stream(vqb_session* s, void* stream) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  CK(cudaSetDevice(s->device));
  CK(cudaStreamSynchronize(s->stream));
  if (s->own_stream) cudaStreamDestroy(s->stream);
  s->stream = reinterpret_cast<cudaStream_t>(stream);
  s->own_stream = false;
  return VQB_OK;
}

int vqb_local_maxabs(vqb_session* s, double* out) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  *out = s->maxabs;
  return VQB_OK;
}

int vqb_session_info(vqb_session* s, int32_t* info) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  info[0] = s->fast ? 1 : 0;
  info[1] = s->cdim;
  info[2] = s->x64 ? 1 : 0;
  info[3] = s->sums_exact ? 1 : 0;
  info[4] = s->ref_exact ? 1 : 0;
  return VQB_OK;
}

int vqb_local_colstats(vqb_session* s, double* colmax, int32_t* collow) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  for (long long l = 0; l < s->dim; ++l) {
    colmax[l] = s->colmax[(size_t)l];
    collow[l] = s->collow[(size_t)l];
  }
  return VQB_OK;
}

// ---------------------------------------------------------------------------
// training loop
// ---------------------------------------------------------------------------

static int check_config(const vqb_train_config* cfg) {
  const long long t = cfg->target_size;
  if (t < 1 || (t & (t - 1)) != 0)
    return fail(VQB_CONFIG, "codebook size must be a power of two, got %lld", t);
  if (!(cfg->epsilon >= 0)) return fail(VQB_CONFIG, "epsilon must be >= 0, got %g", cfg->epsilon);
  if (!(cfg->delta > 0)) return fail(VQB_CONFIG, "split offset delta must be > 0, got %g", cfg->delta);
  if (cfg->max_iterations_per_level < 1)
    return fail(VQB_CONFIG, "max iterations per level must be >= 1, got %lld",
                (long long)cfg->max_iterations_per_level);
  if (cfg->metric != 0 && cfg->metric != 1)
    return fail(VQB_CONFIG, "unknown distortion metric code %d", cfg->metric);
  if (t > (1LL << 24)) return fail(VQB_CONFIG, "codebook size %lld too large for one device", t);
  return VQB_OK;
}

// Summation mode of the cell sums.  Auto: the two-word fixed-point sums
// (exact, order-free, identical for every GPU count) unless (a) the data's
// column span defeats the two-word grid, or (b) the rows are float64 that
// float32 cannot hold and the set is small enough that the reference's own
// rounding sequence is affordable (kOrderedAutoRows): then the ordered path
// reproduces the reference's ascending-index FP64 sums bit for bit.  The
// ordered path needs the whole set on one device.
constexpr long long kOrderedAutoRows = 1LL << 20;
static bool choose_ordered(const vqb_session* s, int requested) {
  if (requested == 1) return true;
  if (requested == 0) return false;
  if (s->n != s->n_global) return false;
  return !s->sums_exact || (s->x64 != nullptr && s->n <= kOrderedAutoRows);
}

static bool tc_enabled() {
  // VQB_TC=0 (or VQB_ASSIGN=ffma) keeps every pass on the FP32 FFMA kernel
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VQB_TC");
    const char* f = getenv("VQB_ASSIGN");
    v = ((e && strcmp(e, "0") == 0) || (f && strcmp(f, "ffma") == 0)) ? 0 : 1;
  }
  return v == 1;
}

// max over a codebook of |c - mu| (the staged operand's magnitude)
static double codebook_span(const vqb_session* s, const double* codebook, long long size) {
  double mx = 0.0;
  for (long long k = 0; k < size; ++k)
    for (long long l = 0; l < s->dim; ++l) {
      const double v = std::fabs(codebook[k * s->dim + l] - (double)s->mu_host[(size_t)l]);
      mx = v > mx ? v : mx;
    }
  return mx;
}

// Power-of-two scales for the fp16 hi/lo operand split of assign_tc: |y~|
// scaled to <= 2^10 (my bounds |x - mu|), |w| = 2|c~| to <= 2^10 (mw bounds
// |w|), and the norm column to <= 2^14 with a power-of-two A column 2^kn.
// Values outside the assumed bounds are caught on the device (rows are
// re-ranked, codebooks send the pass to the FP32 kernel), never mis-scored.
static void tc_configure(const vqb_session* s, DevState* h, double my, double mw) {
  h->tc_on = 0;
  h->tc_bad = 0;
  if (!s->tcb || !s->fast || !tc_enabled()) return;
  if (!(my > 0) || !(mw > 0) || !std::isfinite(my) || !std::isfinite(mw)) return;
  const int ey = 10 - (int)std::ceil(std::log2(my));
  const int ew = 10 - (int)std::ceil(std::log2(mw));
  if (ey + ew > 90 || ey + ew < -90) return;
  const double nmax = (double)s->dim * (mw / 2) * (mw / 2);
  const int kn = std::max(0, (int)std::ceil(std::log2(std::ldexp(nmax, ey + ew))) - 14);
  if (kn > 15) return;
  h->tc_ey = ey;
  h->tc_ew = ew;
  h->tc_kn = kn;
  h->tc_kmin = 64;
  h->tc_kmax = (int)std::min<long long>(tc_max_size(s->cdim), s->kmax);
  h->tc_on = h->tc_kmax >= h->tc_kmin ? 1 : 0;
}

// (Re)build the rows' operand image when the TC pass is on at a new row
// scale (one pass over x32; sessions whose rows stay resident only).
static int build_row_image(vqb_session* s, const DevState* h) {
  static const bool off = [] {
    const char* e = std::getenv("VQB_TC_IMG");  // 0: always convert in-kernel (A/B timing)
    return e && e[0] == '0';
  }();
  const float* xc = s->args().xc;
  if (off || !s->rows_resident || !xc || !h->tc_on) return VQB_OK;
  if (s->aimg && s->aimg_ey == h->tc_ey) return VQB_OK;
  if (!s->aimg) {
    const long long elems = tc_row_image_elems(s->n, s->cdim);
    const long long qn = (s->n + kTcRows - 1) / kTcRows * kTcRows;
    CK(dalloc(&s->aimg, (size_t)elems));
    CK(dalloc(&s->aq, (size_t)qn));
    CK(cudaMemsetAsync(s->aimg, 0, sizeof(unsigned short) * elems, s->stream));
    CK(cudaMemsetAsync(s->aq, 0, sizeof(float) * qn, s->stream));
  }
  CK(launch_build_row_image(xc, s->mu, s->n, s->cdim, h->tc_ey, s->aimg, s->aq, s->sms, s->stream));
  s->aimg_ey = h->tc_ey;
  return VQB_OK;
}

static double data_span(const vqb_session* s, const double* codebook, long long size) {
  // |x - mu| bound: exact from the session's max |x| when known, else the
  // codebook's span (rows beyond it are flagged on the device)
  double mu_max = 0.0;
  for (float v : s->mu_host) mu_max = std::max(mu_max, (double)std::fabs(v));
  if (s->maxabs > 0 && std::isfinite(s->maxabs)) return s->maxabs + mu_max;
  return codebook ? std::max(codebook_span(s, codebook, size), 1e-30) : 0.0;
}

int vqb_step_begin(vqb_session* s, const vqb_train_config* cfg) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  int rc = check_config(cfg);
  if (rc) return rc;
  CK(cudaSetDevice(s->device));
  rc = s->ensure(cfg->target_size);
  if (rc) return rc;
  s->drained = 0;
  s->hist_raw.clear();
  DevState* h = s->st_host;
  std::memset(h, 0, kStateHeader);
  // fixed-point plan from the column stats every rank agreed on (or this shard's)
  rc = s->plan_fixed(h, cfg->global_colmax, cfg->global_collow);
  if (rc) return rc;
  s->ordered = choose_ordered(s, cfg->ordered);
  if (s->ordered && s->n != s->n_global)
    return fail(VQB_USAGE, "reference-order mode needs the whole training set on one device");
  if (s->ordered) {
    rc = s->ensure_ordered(cfg->target_size);
    if (rc) return rc;
    s->delta_on = false;
  } else {
    rc = s->ensure_delta();
    if (rc) return rc;
  }
  h->target = (int)cfg->target_size;
  h->max_iter = (int)cfg->max_iterations_per_level;
  h->metric = cfg->metric;
  h->eps = cfg->epsilon;
  h->delta = cfg->delta;
  h->n_global = s->n_global;
  {
    // centroids stay in the data's convex hull; a split adds delta per level
    const double my = data_span(s, nullptr, 0);
    tc_configure(s, h, my, 2.0 * (my + 16.0 * cfg->delta));
    if (int rc2 = build_row_image(s, h)) return rc2;
  }
  h->mode = kModeTrain;
  h->ordered = s->ordered ? 1 : 0;
  h->size = 1;
  h->iteration = 1;
  h->td_prev = INFINITY;
  // copy only the header part of the state (history is written on device)
  CK(cudaMemcpyAsync(s->st, h, kStateHeader, cudaMemcpyHostToDevice, s->stream));
  KernelArgs a = s->args();
  CK(launch_clear(a, s->stream));
  if (s->ordered) {
    CK(launch_ordered_update(a, true, s->sms, s->stream));  // column sums in row order
  } else {
    CK(launch_epilogue(a, false, true, true, s->sms, s->stream));
  }
  s->pending_init = true;
  return VQB_OK;
}

int vqb_step_local(vqb_session* s) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  KernelArgs a = s->args();
  if (s->fused_ok) CK(launch_pass_small(a, s->sms, s->stream));
  CK(launch_assign(a, s->fast, s->sms, s->stream));
  if (s->fast) CK(launch_rerank(a, s->sms, s->stream));
  CK(launch_epilogue(a, true, !s->ordered, false, s->sms, s->stream));
  if (s->ordered) CK(launch_ordered_update(a, false, s->sms, s->stream));
  return VQB_OK;
}

int vqb_step_finalize(vqb_session* s) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  KernelArgs a = s->args();
  if (s->pending_init) {
    CK(launch_init_centroid(a, s->fast, s->stream));
    s->pending_init = false;
  } else {
    CK(launch_finalize(a, s->fast, s->stream));
  }
  return VQB_OK;
}

static int upload_codebook(vqb_session* s, const double* codebook, long long size);
static int set_state(vqb_session* s, int mode, long long size, int metric, int ordered,
                     const double* codebook = nullptr, const double* gmax = nullptr,
                     const int* glow = nullptr);

// ---- fixed-codebook Lloyd passes over shards (update_codebook after
// assign_cells at one size, the multi-GPU bench step): begin stages the
// codebook with the common fixed-point scale; each pass is lloyd_local ->
// caller allreduces the exchange buffer -> vqb_step_finalize (centroids of
// the combined sums become the current codebook on every rank).
extern "C" int vqb_lloyd_begin(vqb_session* s, const double* codebook, int64_t size,
                               const double* global_colmax, const int32_t* global_collow) {
  if (!s) return fail(VQB_USAGE, "null session");
  if (size < 1) return fail(VQB_USAGE, "codebook must be at least 1x1");
  std::lock_guard<std::recursive_mutex> lock(s->lock_mu);
  CK(cudaSetDevice(s->device));
  int rc = upload_codebook(s, codebook, size);
  if (rc) return rc;
  // one fixed-point plan on every rank (the column stats they agreed on)
  rc = set_state(s, kModeLloydStep, size, 0, 0, codebook, global_colmax, global_collow);
  if (rc) return rc;
  s->ordered = choose_ordered(s, -1);
  if (s->ordered) {
    rc = s->ensure_ordered(size);
    if (rc) return rc;
    s->st_host->ordered = 1;
    CK(cudaMemcpyAsync(&s->st->ordered, &s->st_host->ordered, sizeof(int), cudaMemcpyHostToDevice, s->stream));
  }
  s->lloyd_size = size;
  s->delta_on = false;  // a stateless pass: every row is summed
  s->pending_init = false;
  KernelArgs a = s->args();
  CK(launch_clear(a, s->stream));
  if (s->fast) CK(launch_prep_codebook(a, s->stream));
  return VQB_OK;
}

extern "C" int vqb_lloyd_local(vqb_session* s) {
  if (!s || s->lloyd_size < 1) return fail(VQB_USAGE, "vqb_lloyd_begin first");
  std::lock_guard<std::recursive_mutex> lock(s->lock_mu);
  CK(launch_reset(s->st, kModeLloydStep, (int)s->lloyd_size, 0, s->ordered ? 1 : 0, 1, s->stream));
  return vqb_step_local(s);
}

int vqb_session::batch_graph(int batch) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("VQB_GRAPH");
    enabled = (e && strcmp(e, "0") == 0) ? 0 : 1;
  }
  if (!enabled || !own_stream) return VQB_OK;  // a caller's stream: plain launches
  const int key = (fast ? 1 : 0) | (ordered ? 2 : 0) | (fused_ok ? 4 : 0) | (delta_on ? 8 : 0) | (batch << 4);
  if (graph && graph_kmax == kmax && graph_key == key) return VQB_OK;
  drop_graph();
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
  int rc = VQB_OK;
  for (int i = 0; i < batch && rc == VQB_OK; ++i) {
    rc = vqb_step_local(this);
    if (rc == VQB_OK) rc = vqb_step_finalize(this);
  }
  cudaError_t e = cudaStreamEndCapture(stream, &g);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  CK(e);
  e = cudaGraphInstantiate(&graph, g, 0);
  cudaGraphDestroy(g);
  CK(e);
  graph_kmax = kmax;
  graph_key = key;
  return VQB_OK;
}

int vqb_step_exchange(vqb_session* s, int64_t** device_words, int64_t* count) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  *device_words = reinterpret_cast<int64_t*>(s->ex);
  *count = s->args().ex.words();
  return VQB_OK;
}

int vqb_step_poll(vqb_session* s, int* done) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  CK(cudaMemcpyAsync(s->done_host, &s->st->done, 2 * sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  *done = s->done_host[0];
  return s->drain_hist(s->done_host[1]);
}

int vqb_step_result(vqb_session* s, double* codebook_out, vqb_level_iteration* hist,
                    int64_t hist_cap, int64_t* warn_sizes, int64_t warn_cap, double* final_dists,
                    vqb_train_summary* summary) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock(s->lock_mu);
  CK(cudaSetDevice(s->device));
  CK(cudaStreamSynchronize(s->stream));
  DevState* h = s->st_host;
  CK(cudaMemcpy(h, s->st, kStateHeader, cudaMemcpyDeviceToHost));
  if (!h->done) return fail(VQB_INTERNAL, "training loop has not finished");
  s->delta_on = false;  // the running sums belong to the finished design
  const long long nh = h->n_hist;
  if (int rc = s->drain_hist(nh)) return rc;
  const std::vector<HistRec>& recs = s->hist_raw;
  const long long size = h->size;
  if (codebook_out)
    CK(cudaMemcpy(codebook_out, s->cb[h->cur], sizeof(double) * size * s->dim,
                  cudaMemcpyDeviceToHost));
  if (final_dists) CK(cudaMemcpy(final_dists, s->dists, sizeof(double) * s->n, cudaMemcpyDeviceToHost));
  s->hist_host.resize((size_t)nh);
  for (long long i = 0; i < nh; ++i) {
    vqb_level_iteration& r = s->hist_host[(size_t)i];
    r.codebook_size = recs[(size_t)i].size;
    r.iteration = recs[(size_t)i].iteration;
    r.td = recs[(size_t)i].td;
    r.empty_cells = recs[(size_t)i].empty;
    r.seconds = (double)(recs[(size_t)i].t_ns - h->t0_ns) * 1e-9;
    if (hist && i < hist_cap) hist[i] = r;
  }
  for (long long i = 0; i < std::min<long long>(h->n_warn, kMaxWarn) && i < warn_cap; ++i)
    warn_sizes[i] = h->warn_sizes[i];
  if (summary) {
    summary->total = h->total;
    summary->n_hist = h->n_hist;
    summary->n_warn = h->n_warn;
    summary->passes = h->passes;
    summary->flagged_rows = h->flagged_total;
    summary->flagged_full = h->flagged2_total;
    summary->evals = h->evals;
    summary->final_size = size;
    summary->fast_path = s->fast ? 1 : 0;
    summary->ordered = s->ordered ? 1 : 0;
    summary->sums_exact = s->sums_exact ? 1 : 0;
    summary->ref_exact = s->ref_exact ? 1 : 0;
  }
  return VQB_OK;
}

int vqb_step_history(vqb_session* s, vqb_level_iteration* hist, int64_t cap, int64_t* count) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock(s->lock_mu);
  const long long nh = (long long)s->hist_host.size();
  for (long long i = 0; i < nh && i < cap; ++i) hist[i] = s->hist_host[(size_t)i];
  if (count) *count = nh;
  return VQB_OK;
}

int vqb_train(vqb_session* s, const vqb_train_config* cfg, double* codebook_out,
              vqb_level_iteration* hist, int64_t hist_cap, int64_t* warn_sizes, int64_t warn_cap,
              double* final_dists, vqb_train_summary* summary) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  if (s->n != s->n_global)
    return fail(VQB_USAGE, "vqb_train drives one device; use the vqb_step_* loop for shards");
  int rc = vqb_step_begin(s, cfg);
  if (rc) return rc;
  rc = vqb_step_finalize(s);  // global centroid + first split
  if (rc) return rc;
  // one device holds every row: small-codebook passes run as one fused kernel
  s->fused_ok = s->fast && !s->ordered && s->n == s->n_global;
  struct Reset {
    vqb_session* s;
    ~Reset() { s->fused_ok = false; }
  } reset_fused{s};
  // Speculative batches: passes early-exit on the device once `done` is set,
  // so the host only checks the flag of the previous batch while the next
  // one is already queued (the GPU never waits on the host).
  static const int batch = [] {  // passes per captured graph (VQB_BATCH, default 4)
    const char* e = getenv("VQB_BATCH");
    const int v = e ? atoi(e) : 4;
    return v >= 1 && v <= 64 ? v : 4;
  }();
  long long issued = 0;
  int b = 0;
  const long long max_passes = (long long)(std::log2((double)cfg->target_size) + 1) *
                                   (cfg->max_iterations_per_level + 1) + 8;
  // One batch of passes is captured once into a CUDA graph (every kernel reads
  // its size / mode from the device state, so the same graph serves every
  // level) and relaunched per batch: one host call instead of ~12 launches
  // per pass, which is what bounds the small-codebook levels.
  rc = s->batch_graph(batch);
  if (rc) return rc;
  while (true) {
    if (s->graph) {
      CK(cudaGraphLaunch(s->graph, s->stream));
    } else {
      for (int i = 0; i < batch; ++i) {
        rc = vqb_step_local(s);
        if (rc) return rc;
        rc = vqb_step_finalize(s);
        if (rc) return rc;
      }
    }
    issued += batch;
    // {done, n_hist} of this batch, read once the batch has run
    CK(cudaMemcpyAsync(&s->done_host[2 * b], &s->st->done, 2 * sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaEventRecord(s->ev_batch[b], s->stream));
    if (issued > batch) {
      CK(cudaEventSynchronize(s->ev_batch[b ^ 1]));
      rc = s->drain_hist(s->done_host[2 * (b ^ 1) + 1]);
      if (rc) return rc;
      if (s->done_host[2 * (b ^ 1)]) break;
    }
    if (issued > max_passes + 2 * batch) {
      CK(cudaStreamSynchronize(s->stream));
      if (s->done_host[2 * b]) break;
      return fail(VQB_INTERNAL, "training loop did not terminate after %lld passes", issued);
    }
    b ^= 1;
  }
  return vqb_step_result(s, codebook_out, hist, hist_cap, warn_sizes, warn_cap, final_dists, summary);
}

// ---------------------------------------------------------------------------
// one-shot calls on a session
// ---------------------------------------------------------------------------

static int upload_codebook(vqb_session* s, const double* codebook, long long size) {
  int rc = s->ensure(size);
  if (rc) return rc;
  const size_t bytes = sizeof(double) * size * s->dim;
  char* p = s->pin_alloc(bytes);
  if (p) {  // through the pinned arena: an asynchronous DMA, no pageable staging
    std::memcpy(p, codebook, bytes);
    CK(cudaMemcpyAsync(s->cb[0], p, bytes, cudaMemcpyHostToDevice, s->stream));
  } else {
    CK(cudaMemcpyAsync(s->cb[0], codebook, bytes, cudaMemcpyHostToDevice, s->stream));
  }
  return VQB_OK;
}

static int set_state(vqb_session* s, int mode, long long size, int metric, int ordered,
                     const double* codebook, const double* gmax, const int* glow) {
  DevState* h = s->st_host;
  // configuration fields are written by the reset kernel + this header copy
  std::memset(h, 0, kStateHeader);
  h->target = (int)size;
  h->max_iter = 1;
  h->metric = metric;
  if (int rc = s->plan_fixed(h, gmax, glow)) return rc;
  h->n_global = s->n_global;
  h->mode = mode;
  h->ordered = ordered;
  h->size = (int)size;
  h->iteration = 1;
  h->td_prev = INFINITY;
  if (codebook) {
    tc_configure(s, h, data_span(s, codebook, size), 2.0 * codebook_span(s, codebook, size));
    if (int rc = build_row_image(s, h)) return rc;
  }
  CK(cudaMemcpyAsync(s->st, h, kStateHeader, cudaMemcpyHostToDevice, s->stream));
  return VQB_OK;
}

int vqb_assign(vqb_session* s, const double* codebook, int64_t size, int metric, int64_t* cells64,
               uint32_t* idx32, double* dists, double* total) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  if (size < 1) return fail(VQB_USAGE, "codebook must be at least 1x1");
  if (size > (1LL << 30)) return fail(VQB_USAGE, "codebook too large");
  CK(cudaSetDevice(s->device));
  int rc = upload_codebook(s, codebook, size);
  if (rc) return rc;
  // in-order distortion (sum_inorder) when it is cheap: assign_cells returns
  // the chunk total accumulated in input order (core.py:315-316)
  const int ordered_td = (s->n == s->n_global && s->n <= (1LL << 20)) ? 1 : 0;
  rc = set_state(s, kModeAssignOnly, size, metric, ordered_td, codebook);
  if (rc) return rc;
  KernelArgs a = s->args();
  CK(launch_clear(a, s->stream));
  if (s->fast) CK(launch_prep_codebook(a, s->stream));
  CK(launch_assign(a, s->fast, s->sms, s->stream));
  if (s->fast) CK(launch_rerank(a, s->sms, s->stream));
  CK(launch_epilogue(a, true, false, false, s->sms, s->stream));
  CK(launch_finalize(a, false, s->stream));
  std::vector<int> tmp;
  if (cells64 || idx32) {
    if (idx32) {
      CK(cudaMemcpyAsync(idx32, s->idx, sizeof(int) * s->n, cudaMemcpyDeviceToHost, s->stream));
    } else {
      tmp.resize((size_t)s->n);
      CK(cudaMemcpyAsync(tmp.data(), s->idx, sizeof(int) * s->n, cudaMemcpyDeviceToHost, s->stream));
    }
  }
  if (dists) CK(cudaMemcpyAsync(dists, s->dists, sizeof(double) * s->n, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(s->st_host, s->st, kStateHeader, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (cells64) {
    if (idx32)
      for (long long i = 0; i < s->n; ++i) cells64[i] = idx32[i];
    else
      for (long long i = 0; i < s->n; ++i) cells64[i] = tmp[(size_t)i];
  }
  if (total) *total = s->st_host->total;
  return VQB_OK;
}

int vqb_update(vqb_session* s, const int64_t* cells, const double* old_codebook, int64_t size,
               double* new_codebook, int64_t* counts, int64_t* n_empty) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  CK(cudaSetDevice(s->device));
  int rc = upload_codebook(s, old_codebook, size);
  if (rc) return rc;
  const int ordered = choose_ordered(s, -1) ? 1 : 0;
  rc = set_state(s, kModeUpdateOnly, size, 0, ordered);
  if (rc) return rc;
  if (ordered) {
    rc = s->ensure_ordered(size);
    if (rc) return rc;
  }
  // cells (int64) staged through the dists buffer, narrowed on the device
  CK(cudaMemcpyAsync(s->dists, cells, sizeof(int64_t) * s->n, cudaMemcpyHostToDevice, s->stream));
  CK(launch_cells_to_idx(reinterpret_cast<const long long*>(s->dists), s->idx, s->n, s->sms, s->stream));
  KernelArgs a = s->args();
  CK(launch_clear(a, s->stream));
  if (ordered)
    CK(launch_ordered_update(a, false, s->sms, s->stream));
  else
    CK(launch_epilogue(a, false, true, false, s->sms, s->stream));
  CK(launch_finalize(a, false, s->stream));
  std::vector<long long> hc((size_t)size);
  CK(cudaMemcpyAsync(new_codebook, s->cb[1], sizeof(double) * size * s->dim, cudaMemcpyDeviceToHost,
                     s->stream));
  CK(cudaMemcpyAsync(hc.data(), s->ex + s->kmax * s->dim, sizeof(long long) * size,
                     cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(s->st_host, s->st, kStateHeader, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (counts)
    for (long long i = 0; i < size; ++i) counts[i] = hc[(size_t)i];
  if (n_empty) *n_empty = s->st_host->last_empty;
  return VQB_OK;
}

// ---------------------------------------------------------------------------
// kernel surface (stateless, host buffers)
// ---------------------------------------------------------------------------

int vqb_assign_range(const double* vectors, int64_t m, int64_t dim, const double* codebook,
                     int64_t size, int64_t start, int64_t stop, int metric, int64_t* out_cells,
                     double* out_dists) {
  if (start < 0 || stop > m || start > stop) return fail(VQB_USAGE, "bad row range");
  if (stop == start) return VQB_OK;
  vqb_session* s = nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  int rc = vqb_open(nullptr, vectors + start * dim, stop - start, dim, 0, stop - start, dev, &s);
  if (rc) return rc;
  std::unique_ptr<vqb_session> guard(s);
  return vqb_assign(s, codebook, size, metric, out_cells + start, nullptr, out_dists + start, nullptr);
}

int vqb_update_rows(const double* vectors, int64_t m, int64_t dim, const int64_t* cells,
                    const double* old_codebook, int64_t size, int64_t worker, int64_t stride,
                    double* out_codebook, int64_t* out_counts) {
  if (stride < 1 || worker < 0) return fail(VQB_USAGE, "bad worker/stride");
  if (m < 1) {
    for (long long i = worker; i < size; i += stride) {
      out_counts[i] = 0;
      for (long long l = 0; l < dim; ++l) out_codebook[i * dim + l] = old_codebook[i * dim + l];
    }
    return VQB_OK;
  }
  vqb_session* s = nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  int rc = vqb_open(nullptr, vectors, m, dim, 0, m, dev, &s);
  if (rc) return rc;
  std::unique_ptr<vqb_session> guard(s);
  std::vector<double> nb((size_t)(size * dim));
  std::vector<int64_t> cnt((size_t)size);
  int64_t empty = 0;
  rc = vqb_update(s, cells, old_codebook, size, nb.data(), cnt.data(), &empty);
  if (rc) return rc;
  for (long long i = worker; i < size; i += stride) {
    out_counts[i] = cnt[(size_t)i];
    for (long long l = 0; l < dim; ++l) out_codebook[i * dim + l] = nb[(size_t)(i * dim + l)];
  }
  return VQB_OK;
}

int vqb_column_sums(const double* vectors, int64_t m, int64_t dim, double* out) {
  if (m < 1 || dim < 1) return fail(VQB_USAGE, "column sums need a non-empty matrix");
  double *dx = nullptr, *dout = nullptr;
  CK(dalloc(&dx, (size_t)(m * dim)));
  std::unique_ptr<double, decltype(&cudaFree)> g1(dx, &cudaFree);
  CK(dalloc(&dout, (size_t)dim));
  std::unique_ptr<double, decltype(&cudaFree)> g2(dout, &cudaFree);
  CK(cudaMemcpy(dx, vectors, sizeof(double) * m * dim, cudaMemcpyHostToDevice));
  CK(launch_column_sums_ordered(dx, nullptr, m, (int)dim, dout, 0));
  CK(cudaMemcpy(out, dout, sizeof(double) * dim, cudaMemcpyDeviceToHost));
  return VQB_OK;
}

int vqb_sum_inorder(const double* values, int64_t n, double* out) {
  if (n <= 0) {
    *out = 0.0;
    return VQB_OK;
  }
  double *dv = nullptr, *dout = nullptr;
  CK(dalloc(&dv, (size_t)n));
  std::unique_ptr<double, decltype(&cudaFree)> g1(dv, &cudaFree);
  CK(dalloc(&dout, 1));
  std::unique_ptr<double, decltype(&cudaFree)> g2(dout, &cudaFree);
  CK(cudaMemcpy(dv, values, sizeof(double) * n, cudaMemcpyHostToDevice));
  CK(launch_sum_inorder(dv, n, dout, 0));
  CK(cudaMemcpy(out, dout, sizeof(double), cudaMemcpyDeviceToHost));
  return VQB_OK;
}

int vqb_pair_distance(const double* a, const double* b, int64_t dim, int metric, double* out) {
  double* d = nullptr;
  CK(dalloc(&d, (size_t)(2 * dim + 1)));
  std::unique_ptr<double, decltype(&cudaFree)> g(d, &cudaFree);
  CK(cudaMemcpy(d, a, sizeof(double) * dim, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d + dim, b, sizeof(double) * dim, cudaMemcpyHostToDevice));
  CK(launch_pair_distance(d, d + dim, (int)dim, metric, d + 2 * dim, 0));
  CK(cudaMemcpy(out, d + 2 * dim, sizeof(double), cudaMemcpyDeviceToHost));
  return VQB_OK;
}

// ---------------------------------------------------------------------------
// one-shot host-buffer paths (end-to-end)
// ---------------------------------------------------------------------------

namespace {
// cached scratch session for repeated one-shot calls of the same shape
std::mutex g_cache_mu;
struct Cached {
  vqb_session* s = nullptr;
  long long n = 0, dim = 0;
  int device = -1;
};
Cached g_cache;

// the two chunk slots of vqb_encode_f32, kept between calls (same device and
// row width, chunks no longer than `cap` rows); never freed at exit (the
// context is gone by then)
std::mutex g_enc_mu;
struct EncodeSlots {
  vqb_session* slot[2] = {nullptr, nullptr};
  long long dim = 0, cap = 0;
  int device = -1;
};
EncodeSlots g_enc;

int cached_session(long long n, long long dim, int device, vqb_session** out) {
  if (g_cache.s && g_cache.n == n && g_cache.dim == dim && g_cache.device == device) {
    *out = g_cache.s;
    return VQB_OK;
  }
  delete g_cache.s;
  g_cache.s = nullptr;
  // allocate with a dummy (zero) upload; data is copied per call
  std::unique_ptr<vqb_session> s(new vqb_session());
  CK(cudaSetDevice(device));
  s->device = device;
  CK(cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, device));
  if (int rc = s->make_streams()) return rc;
  s->n = s->n_global = n;
  s->dim = dim;
  s->ntiles_global = (n + kTdTile - 1) / kTdTile;
  CK(dalloc(&s->x32, (size_t)(n * dim + 16)));
  CK(dalloc(&s->scratch, 64));
  if (int rc = s->alloc_common()) return rc;
  CK(cudaMemset(s->mu, 0, sizeof(float) * dim));
  s->mu_host.assign((size_t)dim, 0.f);
  s->fast = fast_dim_supported((int)dim);
  s->cdim = s->fast ? (int)dim : 0;
  g_cache.s = s.release();
  g_cache.n = n;
  g_cache.dim = dim;
  g_cache.device = device;
  *out = g_cache.s;
  return VQB_OK;
}

// centre of the FP32 staging: the codebook's column mean (any centre is
// exact after the re-rank; a central one keeps the certified band tight)
int set_centre_from_codebook(vqb_session* s, const double* codebook, long long size) {
  std::vector<double> acc((size_t)s->dim, 0.0);
  for (long long k = 0; k < size; ++k)
    for (long long l = 0; l < s->dim; ++l) acc[(size_t)l] += codebook[k * s->dim + l];
  std::vector<float> mu((size_t)s->dim, 0.f);
  for (long long l = 0; l < s->dim; ++l)
    mu[(size_t)l] = std::isfinite(acc[(size_t)l]) ? (float)(acc[(size_t)l] / (double)size) : 0.f;
  char* p = s->pin_alloc(sizeof(float) * s->dim);
  if (p) {
    std::memcpy(p, mu.data(), sizeof(float) * s->dim);
    CK(cudaMemcpyAsync(s->mu, p, sizeof(float) * s->dim, cudaMemcpyHostToDevice, s->stream));
  } else {
    CK(cudaMemcpy(s->mu, mu.data(), sizeof(float) * s->dim, cudaMemcpyHostToDevice));
  }
  s->mu_host = mu;
  return VQB_OK;
}

// H2D piece size of the host-buffer paths (VQB_PIECE_MB, default 8): the
// candidate pass of piece i runs while piece i+1 is in flight
size_t piece_bytes() {
  static const size_t b = [] {
    const char* e = getenv("VQB_PIECE_MB");
    const long v = e ? atol(e) : 8;
    return (size_t)(v > 0 ? v : 8) << 20;
  }();
  return b;
}

// Enqueue the H2D of `rows` host rows into s->x32 in pieces, each piece's
// max |x| and FP32 candidate pass launched as soon as it lands (the copy of
// piece i+1 overlaps the distance pass of piece i).  For dims without a fast
// path the exact scan runs after the last piece.
int stream_rows_and_assign(vqb_session* s, const KernelArgs& a, const float* x, long long rows) {
  const size_t row_bytes = sizeof(float) * (size_t)s->dim;
  const size_t piece = std::max<size_t>(row_bytes, piece_bytes() / row_bytes * row_bytes);
  CK(launch_colstats_reset(s->cmax, s->clow, (int)s->dim, s->stream));
  CK(upload(s->x32, x, row_bytes * rows, piece, s->copy_stream, s->stream,
            [&](size_t off, size_t len) -> cudaError_t {
              const long long r0 = (long long)(off / row_bytes), r1 = (long long)((off + len) / row_bytes);
              cudaError_t e = launch_colstats(s->x32 + r0 * s->dim, nullptr, r1 - r0, (int)s->dim, s->cmax,
                                              s->clow, s->sms, s->stream);
              if (e != cudaSuccess || !s->fast) return e;
              KernelArgs c = a;
              c.r0 = r0;
              c.r1 = r1;
              return launch_assign(c, true, s->sms, s->stream);
            }));
  if (!s->fast) CK(launch_assign(a, false, s->sms, s->stream));
  return VQB_OK;
}
}  // namespace

namespace {
// VQB_TRACE=1: host timestamps + device event times of the host-buffer paths
struct Trace {
  bool on = false;
  std::chrono::steady_clock::time_point t0;
  std::vector<std::pair<const char*, double>> host;
  std::vector<std::pair<const char*, cudaEvent_t>> dev;
  cudaStream_t s = nullptr;
  explicit Trace(cudaStream_t st) : s(st) {
    const char* e = getenv("VQB_TRACE");
    on = e && e[0] == '1';
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what, bool device = true) {
    if (!on) return;
    host.push_back({what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count()});
    if (device) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
      dev.push_back({what, e});
    }
  }
  ~Trace() {
    if (!on) return;
    cudaStreamSynchronize(s);
    for (auto& h : host) fprintf(stderr, "[trace] host %-18s %8.3f ms\n", h.first, h.second);
    for (size_t i = 1; i < dev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, dev[0].second, dev[i].second);
      fprintf(stderr, "[trace] dev  %-18s %8.3f ms\n", dev[i].first, ms);
    }
    for (auto& d : dev) cudaEventDestroy(d.second);
  }
};
}  // namespace

int vqb_lloyd_step_f32(const float* x, int64_t n, int64_t dim, const double* codebook,
                       int64_t size, int device, double* new_codebook, int64_t* cells_out,
                       double* td, int64_t* n_empty) {
  if (n < 1 || dim < 1 || size < 1) return fail(VQB_USAGE, "Lloyd step needs non-empty rows and codebook");
  std::lock_guard<std::mutex> lock(g_cache_mu);
  vqb_session* s = nullptr;
  int rc = cached_session(n, dim, device, &s);
  if (rc) return rc;
  CK(cudaSetDevice(device));
  s->fast = fast_dim_supported((int)dim);
  rc = s->ensure(size);
  if (rc) return rc;
  rc = s->pin_reserve(2 * sizeof(double) * size * dim + 4096);
  if (rc) return rc;
  s->pin_off = 0;
  Trace tr(s->stream);
  tr.mark("start");
  const size_t row_bytes = sizeof(float) * (size_t)dim;
  const size_t piece = std::max<size_t>(row_bytes, piece_bytes() / row_bytes * row_bytes);
  const bool pinned_x = host_is_pinned(x);
  if (tr.on) fprintf(stderr, "[trace] pinned=%d\n", pinned_x ? 1 : 0);
  // the small uploads (centre, codebook, state) go first: they share the
  // H2D copy engine with the rows and would otherwise queue behind 64 MB
  rc = set_centre_from_codebook(s, codebook, size);
  if (rc) return rc;
  rc = upload_codebook(s, codebook, size);
  if (rc) return rc;
  rc = set_state(s, kModeLloydStep, size, 0, 0, codebook);
  if (rc) return rc;
  size_t npieces = 0;
  if (pinned_x) {
    // the DMA of every piece starts now; the host work below overlaps it
    npieces = (row_bytes * n + piece - 1) / piece;
    while (s->piece_ev.size() < npieces) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      s->piece_ev.push_back(e);
    }
    CK(cudaEventRecord(s->piece_ev[0], s->stream));  // earlier readers of x32 are done
    CK(cudaStreamWaitEvent(s->copy_stream, s->piece_ev[0], 0));
    for (size_t i = 0; i < npieces; ++i) {
      const size_t off = i * piece, len = std::min(piece, row_bytes * n - off);
      CK(cudaMemcpyAsync(reinterpret_cast<char*>(s->x32) + off, reinterpret_cast<const char*>(x) + off, len,
                         cudaMemcpyHostToDevice, s->copy_stream));
      CK(cudaEventRecord(s->piece_ev[i], s->copy_stream));
    }
  }
  tr.mark("copies_enqueued", false);
  KernelArgs a = s->args();
  CK(launch_clear(a, s->stream));
  if (s->fast) CK(launch_prep_codebook(a, s->stream));
  tr.mark("prepped");
  if (pinned_x) {
    CK(launch_colstats_reset(s->cmax, s->clow, (int)dim, s->stream));
    for (size_t i = 0; i < npieces; ++i) {
      const long long r0 = (long long)(i * piece / row_bytes);
      const long long r1 = std::min<long long>(n, (long long)((i + 1) * piece / row_bytes));
      CK(cudaStreamWaitEvent(s->stream, s->piece_ev[i], 0));
      CK(launch_colstats(s->x32 + r0 * dim, nullptr, r1 - r0, (int)dim, s->cmax, s->clow, s->sms, s->stream));
      if (s->fast) {
        KernelArgs c = a;
        c.r0 = r0;
        c.r1 = r1;
        CK(launch_assign(c, true, s->sms, s->stream));
      }
    }
    if (!s->fast) CK(launch_assign(a, false, s->sms, s->stream));
  } else {
    rc = stream_rows_and_assign(s, a, x, n);
    if (rc) return rc;
  }
  tr.mark("assigned");
  // the fixed-point plan of these rows' column stats, on the device
  CK(launch_set_shift(s->st, s->cmax, s->clow, (int)dim, s->n_global, s->cshift, nullptr, s->stream));
  if (s->fast) CK(launch_rerank(a, s->sms, s->stream));
  tr.mark("reranked");
  CK(launch_epilogue(a, true, true, false, s->sms, s->stream));  // distortion + cell sums
  tr.mark("epilogue");
  CK(launch_finalize(a, false, s->stream));
  tr.mark("finalized");
  char* cb_pin = s->pin_alloc(sizeof(double) * size * dim);
  CK(cudaMemcpyAsync(cb_pin ? cb_pin : reinterpret_cast<char*>(new_codebook), s->cb[1],
                     sizeof(double) * size * dim, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(s->st_host, s->st, kStateHeader, cudaMemcpyDeviceToHost, s->stream));
  if (cells_out) {
    long long* wide = reinterpret_cast<long long*>(s->dists);  // dists are consumed by now
    CK(launch_widen_idx(s->idx, wide, n, s->sms, s->stream));
    CK(download(cells_out, wide, sizeof(long long) * n, s->stream));
  }
  CK(cudaStreamSynchronize(s->stream));
  tr.mark("synced", false);
  if (s->st_host->nonfinite) return fail(VQB_USAGE, "training vectors contain non-finite values");
  if (!s->st_host->sums_exact) {
    // the rows' span defeats the two-word grid: redo the update in the
    // reference's order from the cell table already on the device
    rc = s->ensure_ordered(size);
    if (rc) return rc;
    KernelArgs o = s->args();
    CK(launch_reset(s->st, kModeUpdateOnly, (int)size, 0, 1, 0, s->stream));
    CK(launch_ordered_update(o, false, s->sms, s->stream));
    CK(launch_finalize(o, false, s->stream));
    CK(cudaMemcpyAsync(cb_pin ? cb_pin : reinterpret_cast<char*>(new_codebook), s->cb[1],
                       sizeof(double) * size * dim, cudaMemcpyDeviceToHost, s->stream));
    const double td_keep = s->st_host->total;
    CK(cudaMemcpyAsync(s->st_host, s->st, kStateHeader, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    s->st_host->total = td_keep;
  }
  if (cb_pin) std::memcpy(new_codebook, cb_pin, sizeof(double) * size * dim);
  if (td) *td = s->st_host->total;
  if (n_empty) *n_empty = s->st_host->last_empty;
  return VQB_OK;
}

int vqb_encode_f32(const float* x, int64_t n, int64_t dim, const double* codebook, int64_t size,
                   int device, uint32_t* idx_out, double* total) {
  if (n == 0) {
    if (total) *total = 0.0;
    return VQB_OK;
  }
  if (n < 0 || dim < 1 || size < 1) return fail(VQB_USAGE, "encode needs a non-empty codebook");
  CK(cudaSetDevice(device));
  // Two slots, each a session over a chunk of rows; slot c%2 runs chunk c.
  // The H2D of chunk c (in pieces, each piece's candidate pass launched as
  // it lands) overlaps the tail kernels of chunk c-1; chunk c-1's indices
  // are drained while chunk c computes.  The slots are kept between calls of
  // the same row width on the same device (their ~12 allocations and 4
  // pinned buffers cost ~15 ms per call: 17 -> 2 ms for a 2^20-row encode);
  // a call with longer chunks than the slots hold rebuilds them.
  const long long chunk = std::min<long long>(n, 1LL << 22);
  std::lock_guard<std::mutex> enc_lock(g_enc_mu);
  if (!(g_enc.slot[0] && g_enc.slot[1] && g_enc.device == device && g_enc.dim == dim && g_enc.cap >= chunk)) {
    for (auto& p : g_enc.slot) {
      delete p;
      p = nullptr;
    }
    g_enc.cap = 0;
    for (int i = 0; i < 2; ++i) {
      std::unique_ptr<vqb_session> s(new vqb_session());
      s->device = device;
      CK(cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, device));
      if (int rc = s->make_streams()) return rc;
      s->n = s->n_global = chunk;
      s->dim = dim;
      s->ntiles_global = (chunk + kTdTile - 1) / kTdTile;
      CK(dalloc(&s->x32, (size_t)(chunk * dim + 16)));
      CK(dalloc(&s->scratch, 64));
      if (int rc = s->alloc_common()) return rc;
      g_enc.slot[i] = s.release();
    }
    g_enc.device = device;
    g_enc.dim = dim;
    g_enc.cap = chunk;
  }
  vqb_session* const* slot = g_enc.slot;
  for (int i = 0; i < 2; ++i) {
    vqb_session* s = slot[i];
    // (the previous call ended with both streams synchronised)
    s->pin_off = 0;
    s->n = s->n_global = chunk;
    s->maxabs = 0;
    s->fast = fast_dim_supported((int)dim);
    s->cdim = s->fast ? (int)dim : 0;
    int rc = set_centre_from_codebook(s, codebook, size);
    if (rc) return rc;
    rc = upload_codebook(s, codebook, size);
    if (rc) return rc;
  }
  const long long nchunks = (n + chunk - 1) / chunk;
  double* tot_pinned = nullptr;
  CK(cudaMallocHost(reinterpret_cast<void**>(&tot_pinned), sizeof(double) * nchunks));
  std::unique_ptr<double, decltype(&cudaFreeHost)> gp(tot_pinned, &cudaFreeHost);
  auto drain = [&](long long c) -> int {
    vqb_session* s = slot[c & 1];
    const long long r0 = c * chunk;
    const long long rows = std::min(chunk, n - r0);
    CK(download(idx_out + r0, s->idx, sizeof(int) * rows, s->stream));
    return VQB_OK;
  };
  for (long long c = 0; c < nchunks; ++c) {
    vqb_session* s = slot[c & 1];
    const long long r0 = c * chunk;
    const long long rows = std::min(chunk, n - r0);
    s->n = rows;  // last chunk may be short; tiles beyond it stay zero
    KernelArgs a = s->args();
    if (!total) a.dists = nullptr;  // indices only: no per-row distances
    CK(launch_reset(s->st, kModeAssignOnly, (int)size, 0, 0, 0, s->stream));
    CK(launch_clear(a, s->stream));
    if (s->fast) CK(launch_prep_codebook(a, s->stream));
    int rc = stream_rows_and_assign(s, a, x + r0 * dim, rows);
    if (rc) return rc;
    if (s->fast) CK(launch_rerank(a, s->sms, s->stream));
    CK(launch_epilogue(a, total != nullptr, false, false, s->sms, s->stream));
    CK(launch_finalize(a, false, s->stream));
    CK(cudaMemcpyAsync(tot_pinned + c, &s->st->total, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    if (c > 0) {
      rc = drain(c - 1);
      if (rc) return rc;
    }
  }
  int rc = drain(nchunks - 1);
  if (rc) return rc;
  CK(cudaStreamSynchronize(slot[0]->stream));
  CK(cudaStreamSynchronize(slot[1]->stream));
  if (total) {
    double t = 0.0;
    for (long long c = 0; c < nchunks; ++c) t += tot_pinned[c];
    *total = t;
  }
  return VQB_OK;
}

// ---------------------------------------------------------------------------
// bench helper: device-resident Lloyd iterations with per-kernel event timing
// ---------------------------------------------------------------------------

int vqb_bench_iteration(vqb_session* s, const double* codebook, int64_t size, int reps,
                        double* ms_segments, int64_t* flagged) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  CK(cudaSetDevice(s->device));
  int rc = upload_codebook(s, codebook, size);
  if (rc) return rc;
  rc = set_state(s, kModeLloydStep, size, 0, 0, codebook);
  if (rc) return rc;
  // segments: [prep+clear, assign, rerank, epilogue, finalize]
  cudaEvent_t ev[6];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  double acc[5] = {0, 0, 0, 0, 0};
  KernelArgs a = s->args();
  // staging of the first codebook (later passes are staged by apply_kernel,
  // exactly as inside the training loop)
  CK(launch_clear(a, s->stream));
  if (s->fast) CK(launch_prep_codebook(a, s->stream));
  for (int r = 0; r < reps; ++r) {
    // keep iterating on the device: after each update the new codebook
    // becomes current (cur flips), exactly like consecutive Lloyd passes
    CK(cudaEventRecord(ev[0], s->stream));
    CK(launch_reset(s->st, kModeLloydStep, (int)size, 0, 0, 1, s->stream));
    CK(cudaEventRecord(ev[1], s->stream));
    CK(launch_assign(a, s->fast, s->sms, s->stream));
    CK(cudaEventRecord(ev[2], s->stream));
    if (s->fast) CK(launch_rerank(a, s->sms, s->stream));
    CK(cudaEventRecord(ev[3], s->stream));
    CK(launch_epilogue(a, true, true, false, s->sms, s->stream));  // distortion + cell sums
    CK(cudaEventRecord(ev[4], s->stream));
    CK(launch_finalize(a, s->fast, s->stream));
    CK(cudaEventRecord(ev[5], s->stream));
    CK(cudaEventSynchronize(ev[5]));
    float m;
    for (int k = 0; k < 5; ++k) {
      CK(cudaEventElapsedTime(&m, ev[k], ev[k + 1]));
      acc[k] += m;
    }
  }
  long long flt = 0;
  CK(cudaMemcpy(&flt, &s->st->flagged_total, sizeof(long long), cudaMemcpyDeviceToHost));
  for (auto& e : ev) cudaEventDestroy(e);
  for (int k = 0; k < 5; ++k) ms_segments[k] = acc[k] / reps;
  *flagged = flt / reps;
  return VQB_OK;
}

// Time `reps` device-resident allocation passes (assign_cells / encode over
// the session's rows: candidate pass + re-rank + exact distances + tree-order
// distortion) at a fixed codebook.  ms_out = average per pass (CUDA events on
// the session stream); total_out = the last pass's distortion.
int vqb_bench_assign(vqb_session* s, const double* codebook, int64_t size, int reps, double* ms_out,
                     double* total_out, int64_t* flagged) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  if (reps < 1) return fail(VQB_USAGE, "reps must be >= 1");
  CK(cudaSetDevice(s->device));
  int rc = upload_codebook(s, codebook, size);
  if (rc) return rc;
  rc = set_state(s, kModeAssignOnly, size, 0, 0, codebook);
  if (rc) return rc;
  KernelArgs a = s->args();
  CK(launch_clear(a, s->stream));
  if (s->fast) CK(launch_prep_codebook(a, s->stream));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s->stream));
  for (int r = 0; r < reps; ++r) {
    CK(launch_reset(s->st, kModeAssignOnly, (int)size, 0, 0, 1, s->stream));
    CK(launch_assign(a, s->fast, s->sms, s->stream));
    if (s->fast) CK(launch_rerank(a, s->sms, s->stream));
    CK(launch_epilogue(a, true, false, false, s->sms, s->stream));
    CK(launch_finalize(a, false, s->stream));
  }
  CK(cudaEventRecord(e1, s->stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CK(cudaMemcpy(s->st_host, s->st, kStateHeader, cudaMemcpyDeviceToHost));
  *ms_out = ms / reps;
  if (total_out) *total_out = s->st_host->total;
  if (flagged) *flagged = s->st_host->flagged_total / reps;
  return VQB_OK;
}

// Tensor-core probe (tests): raw accumulators D = 2^(ey+ew) v of rows
// [0, 128) against a codebook of `size` (a multiple of 256 that fits the smem
// image) -> dump[128][size]; scales = {ey, ew, kn, tc_on, tc_bad}.
int vqb_debug_tc_tile(vqb_session* s, const double* codebook, int64_t size, float* dump,
                      int32_t* scales) {
  if (!s) return fail(VQB_USAGE, "null session");
  std::lock_guard<std::recursive_mutex> lock_(s->lock_mu);
  if (size % kTcChunk != 0 || size > tc_max_size(s->cdim))
    return fail(VQB_USAGE, "probe needs a codebook size that is a multiple of %d and <= %d", kTcChunk,
                tc_max_size(s->cdim));
  CK(cudaSetDevice(s->device));
  int rc = upload_codebook(s, codebook, size);
  if (rc) return rc;
  rc = set_state(s, kModeAssignOnly, size, 0, 0, codebook);
  if (rc) return rc;
  KernelArgs a = s->args();
  CK(launch_clear(a, s->stream));
  CK(launch_prep_codebook(a, s->stream));
  float* d = nullptr;
  CK(dalloc(&d, (size_t)(kTcRows * size)));
  std::unique_ptr<float, decltype(&cudaFree)> g(d, &cudaFree);
  CK(cudaMemsetAsync(d, 0xff, sizeof(float) * kTcRows * size, s->stream));
  CK(launch_tc_probe(a, d, s->stream));
  CK(cudaMemcpyAsync(dump, d, sizeof(float) * kTcRows * size, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(s->st_host, s->st, kStateHeader, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  scales[0] = s->st_host->tc_ey;
  scales[1] = s->st_host->tc_ew;
  scales[2] = s->st_host->tc_kn;
  scales[3] = s->st_host->tc_on;
  scales[4] = s->st_host->tc_bad;
  return VQB_OK;
}

// Host->device bandwidth of the copy engine: mode 0 = transfer.cpp upload
// (pinned straight / pageable staged), 1 = one plain cudaMemcpy, 2 =
// cudaHostRegister + upload + unregister (the register cost included).
int vqb_bench_upload(const void* src, int64_t bytes, int mode, double* seconds) {
  void* d = nullptr;
  CK(cudaMalloc(&d, (size_t)bytes));
  std::unique_ptr<void, decltype(&cudaFree)> g(d, &cudaFree);
  cudaStream_t cs, ks;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
  auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaSuccess;
  if (mode == 1) {
    e = cudaMemcpy(d, src, (size_t)bytes, cudaMemcpyHostToDevice);
  } else {
    if (mode == 2) e = cudaHostRegister(const_cast<void*>(src), (size_t)bytes, cudaHostRegisterDefault);
    if (e == cudaSuccess) e = upload(d, src, (size_t)bytes, 16u << 20, cs, ks);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ks);
    if (mode == 2) cudaHostUnregister(const_cast<void*>(src));
  }
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamDestroy(cs);
  cudaStreamDestroy(ks);
  CK(e);
  *seconds = std::chrono::duration<double>(t1 - t0).count();
  return VQB_OK;
}

// ---------------------------------------------------------------------------
// data formats either side of the path (imaging.cu): block vectoriser, raster,
// decode, reconstruction distortion.  Stateless, host buffers; device memory
// from the stream-ordered pool (kept cached across calls).
// ---------------------------------------------------------------------------

}  // extern "C"

namespace {

struct OneShot {
  cudaStream_t stream = nullptr, copy = nullptr;
  int device = -1;
  int init(int dev) {
    CK(cudaSetDevice(dev));
    if (device == dev && stream) return VQB_OK;
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, dev));
    unsigned long long keep = ~0ULL;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    device = dev;
    return VQB_OK;
  }
};
std::mutex g_oneshot_mu;
OneShot g_oneshot;

template <typename T>
struct PoolBuf {
  T* p = nullptr;
  cudaStream_t s;
  explicit PoolBuf(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t count) {
    return cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T), s);
  }
  ~PoolBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

int image_args(int64_t images, int64_t height, int64_t width, int64_t block, long long* count) {
  if (images < 1 || height < 1 || width < 1)
    return fail(VQB_USAGE, "image must be at least 1x1, got %lldx%lld", (long long)width, (long long)height);
  if (block < 1) return fail(VQB_USAGE, "block side must be >= 1, got %lld", (long long)block);
  if (block > 4096) return fail(VQB_USAGE, "block side %lld too large", (long long)block);
  *count = ((height + block - 1) / block) * ((width + block - 1) / block) * images;
  return VQB_OK;
}

}  // namespace

extern "C" {

int vqb_pixels_to_blocks(const uint8_t* pixels, int64_t images, int64_t height, int64_t width, int64_t block,
                         int device, double* out64, float* out32) {
  long long count = 0;
  if (int rc = image_args(images, height, width, block, &count)) return rc;
  if ((out64 == nullptr) == (out32 == nullptr)) return fail(VQB_USAGE, "exactly one of out64 / out32 must be given");
  std::lock_guard<std::mutex> lock(g_oneshot_mu);
  if (int rc = g_oneshot.init(device)) return rc;
  cudaStream_t st = g_oneshot.stream;
  const size_t npx = (size_t)(images * height * width), nout = (size_t)count * block * block;
  PoolBuf<unsigned char> px(st);
  PoolBuf<char> out(st);
  CK(px.alloc(npx));
  CK(out.alloc(nout * (out64 ? 8 : 4)));
  CK(upload(px.p, pixels, npx, 16u << 20, g_oneshot.copy, st));
  if (out64)
    CK(launch_pixels_to_blocks_f64(px.p, images, height, width, (int)block, reinterpret_cast<double*>(out.p), st));
  else
    CK(launch_pixels_to_blocks_f32(px.p, images, height, width, (int)block, reinterpret_cast<float*>(out.p), st));
  CK(download(out64 ? static_cast<void*>(out64) : static_cast<void*>(out32), out.p, nout * (out64 ? 8 : 4), st));
  return VQB_OK;
}

int vqb_blocks_to_pixels(const double* vectors, int64_t images, int64_t height, int64_t width, int64_t block,
                         int device, uint8_t* pixels) {
  long long count = 0;
  if (int rc = image_args(images, height, width, block, &count)) return rc;
  std::lock_guard<std::mutex> lock(g_oneshot_mu);
  if (int rc = g_oneshot.init(device)) return rc;
  cudaStream_t st = g_oneshot.stream;
  const size_t npx = (size_t)(images * height * width), nin = (size_t)count * block * block;
  PoolBuf<double> vin(st);
  PoolBuf<unsigned char> px(st);
  CK(vin.alloc(nin));
  CK(px.alloc(npx));
  CK(upload(vin.p, vectors, nin * sizeof(double), 16u << 20, g_oneshot.copy, st));
  CK(launch_blocks_to_pixels(vin.p, nullptr, nullptr, images, height, width, (int)block, px.p, st));
  CK(download(pixels, px.p, npx, st));
  return VQB_OK;
}

int vqb_decode(const uint32_t* indices, int64_t n, const double* codebook, int64_t size, int64_t dim,
               int device, double* out) {
  if (n < 0 || size < 1 || dim < 1) return fail(VQB_USAGE, "decode needs a non-empty codebook");
  if (n == 0) return VQB_OK;
  std::lock_guard<std::mutex> lock(g_oneshot_mu);
  if (int rc = g_oneshot.init(device)) return rc;
  cudaStream_t st = g_oneshot.stream;
  PoolBuf<double> cb(st);
  PoolBuf<unsigned> idx(st);
  PoolBuf<double> rows(st);
  PoolBuf<int> bad(st);
  CK(cb.alloc((size_t)(size * dim)));
  CK(idx.alloc((size_t)n));
  CK(bad.alloc(1));
  // output in pieces of <= 2^27 doubles (1 GiB): device footprint bounded,
  // the gather of piece i+1 overlaps nothing worth mentioning next to its D2H
  const long long piece = std::max<long long>(1, std::min<long long>(n, (1LL << 27) / dim));
  CK(rows.alloc((size_t)(piece * dim)));
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  CK(upload(cb.p, codebook, sizeof(double) * size * dim, 16u << 20, g_oneshot.copy, st));
  CK(upload(idx.p, indices, sizeof(unsigned) * n, 16u << 20, g_oneshot.copy, st));
  for (long long r0 = 0; r0 < n; r0 += piece) {
    const long long m = std::min(piece, n - r0);
    CK(launch_decode(idx.p + r0, m, (int)dim, cb.p, size, rows.p, bad.p, st));
    CK(download(out + r0 * dim, rows.p, sizeof(double) * m * dim, st));
  }
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hbad) return fail(VQB_FORMAT, "corrupt stream: index >= codebook size %lld", (long long)size);
  return VQB_OK;
}

int vqb_decode_pixels(const uint32_t* indices, int64_t images, int64_t height, int64_t width, int64_t block,
                      const double* codebook, int64_t size, int device, uint8_t* pixels) {
  long long count = 0;
  if (int rc = image_args(images, height, width, block, &count)) return rc;
  if (size < 1) return fail(VQB_USAGE, "decode needs a non-empty codebook");
  std::lock_guard<std::mutex> lock(g_oneshot_mu);
  if (int rc = g_oneshot.init(device)) return rc;
  cudaStream_t st = g_oneshot.stream;
  const long long dim = block * block;
  PoolBuf<double> cb(st);
  PoolBuf<unsigned> idx(st);
  PoolBuf<unsigned char> px(st);
  PoolBuf<int> bad(st);
  CK(cb.alloc((size_t)(size * dim)));
  CK(idx.alloc((size_t)count));
  CK(px.alloc((size_t)(images * height * width)));
  CK(bad.alloc(1));
  CK(upload(cb.p, codebook, sizeof(double) * size * dim, 16u << 20, g_oneshot.copy, st));
  CK(upload(idx.p, indices, sizeof(unsigned) * count, 16u << 20, g_oneshot.copy, st));
  // the raster reads codebook rows by index: validate the indices first
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  CK(launch_index_check(idx.p, count, size, bad.p, st));
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hbad) return fail(VQB_FORMAT, "corrupt stream: index >= codebook size %lld", (long long)size);
  PoolBuf<unsigned char> cbq(st);
  CK(cbq.alloc((size_t)(size * dim)));
  CK(launch_decode_pixels(idx.p, cb.p, size, images, height, width, (int)block, cbq.p, px.p, st));
  CK(download(pixels, px.p, (size_t)(images * height * width), st));
  return VQB_OK;
}

int vqb_reconstruction_distortion(const double* a, const double* b, int64_t n, int64_t dim, int metric,
                                  int device, double* total) {
  if (n < 0 || dim < 1) return fail(VQB_USAGE, "dimension must be >= 1");
  if (metric != kSquared && metric != kEuclidean) return fail(VQB_USAGE, "unknown metric code %d", metric);
  if (n == 0) {
    *total = 0.0;
    return VQB_OK;
  }
  std::lock_guard<std::mutex> lock(g_oneshot_mu);
  if (int rc = g_oneshot.init(device)) return rc;
  cudaStream_t st = g_oneshot.stream;
  PoolBuf<double> da(st), db(st), d(st), tiles(st), out(st);
  CK(da.alloc((size_t)(n * dim)));
  CK(db.alloc((size_t)(n * dim)));
  CK(d.alloc((size_t)n));
  CK(tiles.alloc((size_t)((n + kTdTile - 1) / kTdTile)));
  CK(out.alloc(1));
  const size_t row_bytes = sizeof(double) * (size_t)dim;
  const size_t piece = std::max<size_t>(row_bytes, ((size_t)16 << 20) / row_bytes * row_bytes);
  CK(upload(da.p, a, row_bytes * n, piece, g_oneshot.copy, st));
  // per-row distances of each piece of b as it lands
  CK(upload(db.p, b, row_bytes * n, piece, g_oneshot.copy, st, [&](size_t off, size_t len) -> cudaError_t {
    const long long r0 = (long long)(off / row_bytes), r1 = (long long)((off + len) / row_bytes);
    return launch_pair_rows(da.p + r0 * dim, db.p + r0 * dim, r1 - r0, (int)dim, metric, d.p + r0, st);
  }));
  // sum_inorder (_kernels.py:92-98) for up to 2^20 rows; above, the fixed tree
  // of 2048-row tiles (the training loop's distortion order)
  CK(launch_distortion_sum(d.p, n, n <= (1LL << 20), tiles.p, out.p, st));
  CK(cudaMemcpyAsync(total, out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return VQB_OK;
}

// Device-resident timing of one imaging kernel (bench.py --workload formats):
// which = 0 pixels_to_blocks f32, 1 pixels_to_blocks f64, 2 blocks_to_pixels,
// 3 decode (n rows of dim from a size-row codebook), 4 decode_pixels,
// 5 per-row pair distances (n x dim).  Inputs are synthetic device buffers;
// ms_out = mean event time per launch over `reps`, bytes_out = algorithmic
// bytes per launch (every input byte read once, every output byte written once).
int vqb_bench_formats(int which, int64_t images, int64_t height, int64_t width, int64_t block, int64_t n,
                      int64_t dim, int64_t size, int reps, double* ms_out, double* bytes_out) {
  if (reps < 1) return fail(VQB_USAGE, "reps must be >= 1");
  long long count = 0;
  if (which <= 2 || which == 4) {
    if (int rc = image_args(images, height, width, block, &count)) return rc;
    dim = block * block;
    n = count;
  }
  if (n < 1 || dim < 1 || size < 1) return fail(VQB_USAGE, "empty benchmark shape");
  std::lock_guard<std::mutex> lock(g_oneshot_mu);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (int rc = g_oneshot.init(dev)) return rc;
  cudaStream_t st = g_oneshot.stream;
  const long long npx = images * height * width;
  PoolBuf<unsigned char> px(st);
  PoolBuf<double> vec(st), vec2(st), cb(st), d(st);
  PoolBuf<float> vec32(st);
  PoolBuf<unsigned> idx(st);
  PoolBuf<int> bad(st);
  PoolBuf<unsigned char> cbq(st);
  double bytes = 0;
  CK(bad.alloc(1));
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  switch (which) {
    case 0: case 1: case 2:
      CK(px.alloc((size_t)npx));
      CK(cudaMemsetAsync(px.p, 0x5a, (size_t)npx, st));
      if (which == 0) {
        CK(vec32.alloc((size_t)(n * dim)));
        bytes = (double)npx + 4.0 * n * dim;
      } else {
        CK(vec.alloc((size_t)(n * dim)));
        CK(cudaMemsetAsync(vec.p, 0, sizeof(double) * n * dim, st));
        bytes = (double)npx + 8.0 * n * dim;
      }
      break;
    case 3: case 4:
      CK(cb.alloc((size_t)(size * dim)));
      CK(cudaMemsetAsync(cb.p, 0, sizeof(double) * size * dim, st));
      CK(idx.alloc((size_t)n));
      CK(cudaMemsetAsync(idx.p, 0, sizeof(unsigned) * n, st));  // index 0: valid
      if (which == 3) {
        CK(vec.alloc((size_t)(n * dim)));
        bytes = 4.0 * n + 8.0 * n * dim;
      } else {
        CK(px.alloc((size_t)npx));
        CK(cbq.alloc((size_t)(size * dim)));
        bytes = 4.0 * n + (double)npx;
      }
      break;
    case 5:
      CK(vec.alloc((size_t)(n * dim)));
      CK(vec2.alloc((size_t)(n * dim)));
      CK(d.alloc((size_t)n));
      CK(cudaMemsetAsync(vec.p, 0, sizeof(double) * n * dim, st));
      CK(cudaMemsetAsync(vec2.p, 0, sizeof(double) * n * dim, st));
      bytes = 16.0 * n * dim + 8.0 * n;
      break;
    default:
      return fail(VQB_USAGE, "unknown kernel %d", which);
  }
  auto launch = [&]() -> cudaError_t {
    switch (which) {
      case 0: return launch_pixels_to_blocks_f32(px.p, images, height, width, (int)block, vec32.p, st);
      case 1: return launch_pixels_to_blocks_f64(px.p, images, height, width, (int)block, vec.p, st);
      case 2: return launch_blocks_to_pixels(vec.p, nullptr, nullptr, images, height, width, (int)block, px.p, st);
      case 3: return launch_decode(idx.p, n, (int)dim, cb.p, size, vec.p, bad.p, st);
      case 4: return launch_decode_pixels(idx.p, cb.p, size, images, height, width, (int)block, cbq.p, px.p, st);
      default: return launch_pair_rows(vec.p, vec2.p, n, (int)dim, 0, d.p, st);
    }
  };
  CK(launch());  // warm-up
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  for (int r = 0; r < reps; ++r) CK(launch());
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms_out = ms / reps;
  *bytes_out = bytes;
  return VQB_OK;
}

int vqb_split_codebook(const double* codebook, int64_t size, int64_t dim, double delta, int device,
                       double* out) {
  if (size < 1 || dim < 1) return fail(VQB_USAGE, "codebook must be at least 1x1");
  if (!(delta > 0)) return fail(VQB_CONFIG, "split offset delta must be > 0, got %g", delta);
  std::lock_guard<std::mutex> lock(g_oneshot_mu);
  if (int rc = g_oneshot.init(device)) return rc;
  cudaStream_t st = g_oneshot.stream;
  PoolBuf<double> cb(st), o(st);
  CK(cb.alloc((size_t)(size * dim)));
  CK(o.alloc((size_t)(2 * size * dim)));
  CK(cudaMemcpyAsync(cb.p, codebook, sizeof(double) * size * dim, cudaMemcpyHostToDevice, st));
  CK(launch_split_rows(cb.p, size, (int)dim, delta, o.p, st));
  CK(cudaMemcpyAsync(out, o.p, sizeof(double) * 2 * size * dim, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return VQB_OK;
}

}  // extern "C"
