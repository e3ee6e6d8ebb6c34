// Host<->device copy engine for the host-buffer entry points (vqb_open,
// vqb_encode_f32, vqb_lloyd_step_f32).
//
// * Pinned (page-locked) host buffers go straight to the DMA engine.
// * Pageable buffers -- what a numpy caller hands us -- are staged through a
//   ring of pinned buffers that a small pool of host threads fills with
//   parallel memcpy, so host copying of chunk i+1 overlaps the DMA of chunk i
//   and the PCIe link stays busy (a single-threaded pageable cudaMemcpy runs
//   at a fraction of the link rate).
// * Every chunk is a separate cudaMemcpyAsync on a copy stream followed by an
//   event the compute stream waits on, so kernels that consume chunk i can
//   start while chunk i+1 is still in flight (the caller's `after` hook).
#include "transfer.h"

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace vqb {

namespace {

// -------------------------------------------------------------------------
// a tiny persistent thread pool for parallel memcpy
// -------------------------------------------------------------------------
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }

  // memcpy split over the pool's threads (plus the caller); blocks until done
  void copy(void* dst, const void* src, size_t bytes) {
    const int parts = (int)std::min<size_t>(workers_.size() + 1, std::max<size_t>(1, bytes >> 20));
    if (parts <= 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    const size_t step = (bytes + parts - 1) / parts;
    {
      std::unique_lock<std::mutex> lk(mu_);
      for (int p = 1; p < parts; ++p) {
        const size_t off = std::min(bytes, (size_t)p * step);
        const size_t len = std::min(step, bytes - off);
        jobs_.push_back({static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len});
      }
      pending_ += parts - 1;
    }
    cv_.notify_all();
    std::memcpy(dst, src, std::min(step, bytes));
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  struct Job {
    char* dst;
    const char* src;
    size_t len;
  };

  CopyPool() {
    unsigned hw = std::thread::hardware_concurrency();
    int n = (int)std::min(7u, hw > 1 ? hw - 1 : 1u);
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { run(); });
  }
  ~CopyPool() {
    {
      std::unique_lock<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

  void run() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
        if (stop_ && jobs_.empty()) return;
        j = jobs_.back();
        jobs_.pop_back();
      }
      std::memcpy(j.dst, j.src, j.len);
      {
        std::unique_lock<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_all();
      }
    }
  }

  std::vector<std::thread> workers_;
  std::vector<Job> jobs_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  int pending_ = 0;
  bool stop_ = false;
};

// pinned staging ring shared by all uploads of the process (serialised)
struct StagingRing {
  static constexpr int kBuffers = 3;
  static constexpr size_t kBytes = 16u << 20;
  char* buf[kBuffers] = {nullptr, nullptr, nullptr};
  cudaEvent_t free_ev[kBuffers] = {nullptr, nullptr, nullptr};
  int device = -1;
  std::mutex mu;

  cudaError_t ensure(int dev) {
    if (device == dev && buf[0]) return cudaSuccess;
    release();
    for (int i = 0; i < kBuffers; ++i) {
      cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&buf[i]), kBytes);
      if (e != cudaSuccess) return e;
      e = cudaEventCreateWithFlags(&free_ev[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    device = dev;
    return cudaSuccess;
  }
  void release() {
    for (int i = 0; i < kBuffers; ++i) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (free_ev[i]) cudaEventDestroy(free_ev[i]);
      buf[i] = nullptr;
      free_ev[i] = nullptr;
    }
    device = -1;
  }
};

StagingRing& ring() {
  static StagingRing r;
  return r;
}

}  // namespace

bool host_is_pinned(const void* p) {
  cudaPointerAttributes attr{};
  cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

void host_parallel_copy(void* dst, const void* src, size_t bytes) { CopyPool::get().copy(dst, src, bytes); }

cudaError_t upload(void* dst, const void* src, size_t bytes, size_t chunk, cudaStream_t copy_stream,
                   cudaStream_t compute_stream, const std::function<cudaError_t(size_t, size_t)>& after) {
  if (bytes == 0) return cudaSuccess;
  if (chunk == 0) chunk = bytes;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const bool pinned = host_is_pinned(src);
  std::unique_lock<std::mutex> lk(ring().mu, std::defer_lock);
  if (!pinned) {
    lk.lock();
    e = ring().ensure(dev);
    if (e != cudaSuccess) return e;
    chunk = std::min(chunk, StagingRing::kBytes);
  }
  cudaEvent_t ev;
  e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e != cudaSuccess) return e;
  // the copy stream must not run ahead of earlier work on the compute stream
  // that still reads `dst`
  e = cudaEventRecord(ev, compute_stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(copy_stream, ev, 0);
  int b = 0;
  for (size_t off = 0; off < bytes && e == cudaSuccess; off += chunk) {
    const size_t len = std::min(chunk, bytes - off);
    char* d = static_cast<char*>(dst) + off;
    const char* s = static_cast<const char*>(src) + off;
    if (pinned) {
      e = cudaMemcpyAsync(d, s, len, cudaMemcpyHostToDevice, copy_stream);
    } else {
      StagingRing& r = ring();
      e = cudaEventSynchronize(r.free_ev[b]);  // the DMA out of this buffer is done
      if (e != cudaSuccess) break;
      host_parallel_copy(r.buf[b], s, len);
      e = cudaMemcpyAsync(d, r.buf[b], len, cudaMemcpyHostToDevice, copy_stream);
      if (e == cudaSuccess) e = cudaEventRecord(r.free_ev[b], copy_stream);
      b = (b + 1) % StagingRing::kBuffers;
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev, copy_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(compute_stream, ev, 0);
    if (e == cudaSuccess && after) e = after(off, len);
  }
  cudaEventDestroy(ev);
  return e;
}

cudaError_t download(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return cudaSuccess;
  if (host_is_pinned(dst)) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream);
    return e == cudaSuccess ? cudaStreamSynchronize(stream) : e;
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(ring().mu);
  StagingRing& r = ring();
  e = r.ensure(dev);
  if (e != cudaSuccess) return e;
  // D2H into pinned buffer b while the host drains buffer b-1
  const size_t chunk = StagingRing::kBytes;
  const size_t n = (bytes + chunk - 1) / chunk;
  for (size_t i = 0; i <= n && e == cudaSuccess; ++i) {
    if (i < n) {
      const int b = (int)(i % StagingRing::kBuffers);
      const size_t off = i * chunk, len = std::min(chunk, bytes - off);
      e = cudaStreamWaitEvent(stream, r.free_ev[b], 0);  // an upload's DMA may still read it
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(r.buf[b], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                            stream);
      if (e == cudaSuccess) e = cudaEventRecord(r.free_ev[b], stream);
    }
    if (i > 0 && e == cudaSuccess) {
      const size_t j = i - 1;
      const int pb = (int)(j % StagingRing::kBuffers);
      const size_t off = j * chunk, len = std::min(chunk, bytes - off);
      e = cudaEventSynchronize(r.free_ev[pb]);
      if (e == cudaSuccess) host_parallel_copy(static_cast<char*>(dst) + off, r.buf[pb], len);
    }
  }
  return e;
}

}  // namespace vqb

// ---------------------------------------------------------------------------
// host helpers of the Python types (TrainingSet, core.py:72-99): snapshot
// copies and the finiteness check of float32 rows, split over host threads
// ---------------------------------------------------------------------------

#include "../../include/vqb200.h"

extern "C" int vqb_host_copy(void* dst, const void* src, int64_t bytes) {
  if (bytes > 0) vqb::host_parallel_copy(dst, src, (size_t)bytes);
  return VQB_OK;
}

namespace {
template <typename T, typename U, U kExpMask>
int first_nonfinite(const T* x, int64_t n, int64_t* first) {
  *first = -1;
  if (n <= 0) return VQB_OK;
  const unsigned hw = std::thread::hardware_concurrency();
  const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(hw ? hw : 1, n >> 20));
  std::vector<int64_t> found((size_t)parts, -1);
  auto scan = [&](int p) {
    const int64_t lo = n * p / parts, hi = n * (p + 1) / parts;
    const U* u = reinterpret_cast<const U*>(x);
    for (int64_t i = lo; i < hi; ++i)
      if ((u[i] & kExpMask) == kExpMask) {  // exponent all ones: inf or NaN
        found[(size_t)p] = i;
        return;
      }
  };
  std::vector<std::thread> ts;
  for (int p = 1; p < parts; ++p) ts.emplace_back(scan, p);
  scan(0);
  for (auto& t : ts) t.join();
  for (int64_t f : found)
    if (f >= 0) {
      *first = f;
      break;
    }
  return VQB_OK;
}
}  // namespace

extern "C" int vqb_first_nonfinite_f64(const double* x, int64_t n, int64_t* first) {
  return first_nonfinite<double, uint64_t, 0x7ff0000000000000ull>(x, n, first);
}

extern "C" int vqb_first_nonfinite_f32(const float* x, int64_t n, int64_t* first) {
  return first_nonfinite<float, uint32_t, 0x7f800000u>(x, n, first);
}
