// Reference-order cell sums (update_rows, _kernels.py:39-66: the members of
// cell i are added in ascending training index, one FP64 rounding per add)
// in O(N) work per pass:
//
//   ord_count    per (cell, row block) member counts (block-private smem
//                histogram), stored cell-major: obase[k * B + b]
//   scan         exclusive scan of obase -> the first sorted slot of cell k's
//                members that lie in row block b (cell-major = cells in
//                ascending order, blocks in ascending row order)
//   ord_scatter  stable counting sort: one warp per row block walks its rows
//                in order, 32 at a time; lanes holding the same cell get
//                consecutive slots (match.any + rank below the lane)
//   ord_chain    one warp per (cell, 32 dimensions): lane l runs the
//                reference's sequential FP64 chain over the cell's rows in
//                ascending index (loads prefetched 8 rows ahead, the adds in
//                order), then divides by the count or keeps the old row.
//
// The chains are the reference's own rounding sequence, so the centroids are
// bit-identical to update_rows for every input (float64 rows that are not
// float32-exact, or data whose column span defeats the two-word fixed-point
// grid).  Used only on one device holding the whole set (the order spans it).
#include <climits>

#include "ptx.h"
#include "refarith.cuh"
#include "vqb200_internal.h"

namespace vqb {

constexpr int kOrdMinRows = 2048;
constexpr int kOrdMaxBlocks = 1024;
constexpr int kOrdSmemCells = 48 * 1024;  // histogram / base table in smem up to this many cells

int ordered_blocks(long long n) {
  long long r = (n + kOrdMaxBlocks - 1) / kOrdMaxBlocks;
  if (r < kOrdMinRows) r = kOrdMinRows;
  r = (r + 31) / 32 * 32;
  return (int)((n + r - 1) / r);
}

__device__ __forceinline__ long long ord_rows_per_block(long long n, int B) {
  long long r = (n + B - 1) / B;
  return (r + 31) / 32 * 32;
}

__global__ void __launch_bounds__(256) ord_count_kernel(KernelArgs a) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = st->size;
  const int B = a.oblocks;
  const long long R = ord_rows_per_block(a.n, B);
  const long long r0 = blockIdx.x * R;
  const long long r1 = r0 + R < a.n ? r0 + R : a.n;
  extern __shared__ int hist[];
  const bool smem = K <= kOrdSmemCells;
  if (smem) {
    for (int k = threadIdx.x; k < K; k += blockDim.x) hist[k] = 0;
    __syncthreads();
    for (long long r = r0 + threadIdx.x; r < r1; r += blockDim.x) atomicAdd(hist + a.idx[r], 1);
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) a.obase[(long long)k * B + blockIdx.x] = hist[k];
  } else {
    // (the table was zeroed by the scan of the previous pass's launch_ordered_update)
    for (long long r = r0 + threadIdx.x; r < r1; r += blockDim.x)
      atomicAdd(a.obase + (long long)a.idx[r] * B + blockIdx.x, 1);
  }
}

constexpr int kScanChunk = 4096;  // elements per scan block (256 threads x 16)

// phase 1: sum of each chunk
__global__ void __launch_bounds__(256) ord_scan_sums_kernel(KernelArgs a) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const long long total = (long long)st->size * a.oblocks;
  const long long c0 = blockIdx.x * (long long)kScanChunk;
  if (c0 >= total) return;
  long long v = 0;
  for (long long i = c0 + threadIdx.x; i < c0 + kScanChunk && i < total; i += blockDim.x) v += a.obase[i];
  __shared__ long long red[8];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    a.oscan[blockIdx.x] = (int)t;
  }
}

// block-wide exclusive scan of 256 x 16 values held 16 per thread (in place)
__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += warp_tot[w];
  __syncthreads();
  return base + incl - v;
}

// phase 2: exclusive scan of the chunk sums (one block, looped)
__global__ void __launch_bounds__(256) ord_scan_top_kernel(KernelArgs a) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const long long total = (long long)st->size * a.oblocks;
  const int chunks = (int)((total + kScanChunk - 1) / kScanChunk);
  __shared__ int warp_tot[8];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < chunks; c0 += 256) {
    const int i = c0 + threadIdx.x;
    const int v = i < chunks ? a.oscan[i] : 0;
    const int ex = block_exclusive_scan(v, warp_tot);
    const int base = carry;
    if (i < chunks) a.oscan[i] = base + ex;
    __syncthreads();
    if (threadIdx.x == 255) carry = base + ex + v;
    __syncthreads();
  }
}

// phase 3: exclusive scan within each chunk plus the chunk's offset
__global__ void __launch_bounds__(256) ord_scan_apply_kernel(KernelArgs a) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const long long total = (long long)st->size * a.oblocks;
  const long long c0 = blockIdx.x * (long long)kScanChunk;
  if (c0 >= total) return;
  __shared__ int warp_tot[8];
  // thread t owns elements c0 + 16 t .. c0 + 16 t + 15 (contiguous)
  int v[16];
  int sum = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const long long i = c0 + 16LL * threadIdx.x + j;
    v[j] = i < total ? a.obase[i] : 0;
    sum += v[j];
  }
  int run = a.oscan[blockIdx.x] + block_exclusive_scan(sum, warp_tot);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const long long i = c0 + 16LL * threadIdx.x + j;
    if (i < total) a.obase[i] = run;
    run += v[j];
  }
}

// stable scatter: one warp per row block
__global__ void __launch_bounds__(32) ord_scatter_kernel(KernelArgs a) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = st->size;
  const int B = a.oblocks;
  const long long R = ord_rows_per_block(a.n, B);
  const long long r0 = blockIdx.x * R;
  const long long r1 = r0 + R < a.n ? r0 + R : a.n;
  extern __shared__ int base_s[];
  const bool smem = K <= kOrdSmemCells;
  int* base = base_s;
  const int lane = threadIdx.x;
  if (smem) {
    for (int k = lane; k < K; k += 32) base_s[k] = a.obase[(long long)k * B + blockIdx.x];
    __syncwarp();
  }
  const unsigned lt = (1u << lane) - 1u;
  for (long long r = r0; r < r1; r += 32) {
    const long long row = r + lane;
    const bool ok = row < r1;
    const int c = ok ? a.idx[row] : -1;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    const unsigned peers = __match_any_sync(0xffffffffu, c) & act;
    int* slot = smem ? base + c : a.obase + (long long)(c < 0 ? 0 : c) * B + blockIdx.x;
    const int b0 = ok ? *slot : 0;
    __syncwarp();
    if (ok) {
      a.operm[b0 + __popc(peers & lt)] = (int)row;
      if ((peers & lt) == 0) *slot = b0 + __popc(peers);  // the group's lowest lane advances the slot
    }
    __syncwarp();
  }
}

// sequential reference-order chains, one warp per (cell, 32-dimension chunk)
template <typename XT>
__global__ void __launch_bounds__(32) ord_chain_kernel(KernelArgs a, const XT* __restrict__ X, int zero_cells) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = zero_cells ? 1 : st->size;
  const int dim = a.dim;
  const int dchunks = (dim + 31) / 32;
  const int k = blockIdx.x / dchunks;
  const int d = (blockIdx.x % dchunks) * 32 + threadIdx.x;
  if (k >= K) return;
  const int B = a.oblocks;
  long long start = 0, end = a.n;
  if (!zero_cells) {
    start = a.obase[(long long)k * B];
    end = k + 1 < K ? a.obase[(long long)(k + 1) * B] : a.n;
  }
  const long long cnt = end - start;
  const bool on = d < dim;
  double s = 0.0;
  for (long long b = start; b < end; b += 32) {
    const int m = end - b < 32 ? (int)(end - b) : 32;
    const int p = threadIdx.x < m ? (zero_cells ? (int)(b + threadIdx.x) : a.operm[b + threadIdx.x]) : 0;
    for (int j0 = 0; j0 < m; j0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = __shfl_sync(0xffffffffu, p, j0 + u);
        v[u] = (on && j0 + u < m) ? load_x(X, (long long)r * dim + d) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < m) s = __dadd_rn(s, v[u]);
    }
  }
  if (on) {
    const long long i = (long long)k * dim + d;
    a.ord[i] = cnt > 0 ? __ddiv_rn(s, (double)cnt) : a.cb[st->cur][i];
  }
  if (threadIdx.x == 0 && blockIdx.x % dchunks == 0) a.ex.counts()[k] = cnt;
}

cudaError_t launch_ordered_update(const KernelArgs& a, bool zero_cells, int sms, cudaStream_t s) {
  (void)sms;
  cudaError_t e;
  const int B = a.oblocks;
  const long long kmax = zero_cells ? 1 : a.kmax;
  if (!zero_cells) {
    const size_t smem = (size_t)(a.kmax <= kOrdSmemCells ? a.kmax : 0) * sizeof(int);
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(ord_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(ord_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    if (a.kmax > kOrdSmemCells) {
      e = cudaMemsetAsync(a.obase, 0, sizeof(int) * (size_t)a.kmax * B, s);
      if (e != cudaSuccess) return e;
    }
    e = launch_k(ord_count_kernel, B, 256, smem, s, a);
    if (e != cudaSuccess) return e;
    const long long chunks = (a.kmax * B + kScanChunk - 1) / kScanChunk;
    e = launch_k(ord_scan_sums_kernel, (unsigned)chunks, 256, 0, s, a);
    if (e != cudaSuccess) return e;
    e = launch_k(ord_scan_top_kernel, 1, 256, 0, s, a);
    if (e != cudaSuccess) return e;
    e = launch_k(ord_scan_apply_kernel, (unsigned)chunks, 256, 0, s, a);
    if (e != cudaSuccess) return e;
    e = launch_k(ord_scatter_kernel, B, 32, smem, s, a);
    if (e != cudaSuccess) return e;
  }
  const int dchunks = (a.dim + 31) / 32;
  if (a.x32)
    e = launch_k(ord_chain_kernel<float>, (unsigned)(kmax * dchunks), 32, 0, s, a, a.x32, zero_cells ? 1 : 0);
  else
    e = launch_k(ord_chain_kernel<double>, (unsigned)(kmax * dchunks), 32, 0, s, a, a.x64, zero_cells ? 1 : 0);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace vqb
