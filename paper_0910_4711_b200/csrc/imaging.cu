// Block vectoriser, decode and reconstruction distortion on the device: the
// data formats on either side of the LBG path.
//
//  * pixels_to_blocks (storage.py:281-293): uint8 image -> row-major b x b
//    block vectors, ragged edges padded by replication (np.pad mode="edge").
//  * blocks_to_image raster (storage.py:296-311): block vectors -> uint8
//    pixels, clamp to [0,255], floor(v + 0.5), crop the padding.
//  * decode (codec.py:96-114): row j = codebook[indices[j]]; fused with the
//    raster for the image codec (indices -> pixels, no FP64 intermediate).
//  * reconstruction_distortion (codec.py:135-156): per-row pair_distance
//    (_kernels.py:69-78) in the reference arithmetic + the distortion sum.
//
// All of these are HBM-bound byte movers: one CTA per band of b pixel rows,
// the band staged in shared memory so that both the pixel rows and the
// (contiguous) run of block vectors the band produces are read / written with
// coalesced accesses.  The codebook of the decode paths (<= a few MB) lives in
// L2.  Grids are sized to the work (bands x images), grid-stride elsewhere.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "../../include/vqb200.h"
#include "refarith.cuh"
#include "transfer.h"
#include "vqb200_internal.h"

namespace vqb {

namespace {

constexpr int kBandThreads = 256;
constexpr int kBandSmem = 48 * 1024;  // largest staged band (b x padded width bytes)

// ---------------------------------------------------------------------------
// pixels -> block vectors
// ---------------------------------------------------------------------------

// One CTA per (band of B pixel rows, image).  The band's block vectors are the
// contiguous run [band * bcols, (band + 1) * bcols) of the output, so output
// element o of the run is (block bx = o / BB, in-block row r, column c).
template <int B, typename OutT>
__global__ void __launch_bounds__(kBandThreads) pixels_to_blocks_band(
    const unsigned char* __restrict__ px, long long H, long long W, int bcols, int brows,
    OutT* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char band[];  // [B][Wp]
  constexpr int BB = B * B;
  const long long img = blockIdx.y;
  const int by = blockIdx.x;
  const int Wp = bcols * B;
  const unsigned char* src = px + img * H * W;
  if ((W & 15) == 0 && Wp == W) {
    // no right padding, 16-byte aligned rows: one uint4 per thread per row
    const int w16 = (int)(W >> 4);
    for (int v = threadIdx.x; v < B * w16; v += kBandThreads) {
      const int r = v / w16, x16 = v - r * w16;
      const long long y = min((long long)by * B + r, H - 1);  // replicate the bottom edge
      reinterpret_cast<uint4*>(band + r * Wp)[x16] = __ldg(reinterpret_cast<const uint4*>(src + y * W) + x16);
    }
  } else {
    for (int r = 0; r < B; ++r) {
      const long long y = min((long long)by * B + r, H - 1);  // replicate the bottom edge
      const unsigned char* row = src + y * W;
      for (int x = threadIdx.x; x < Wp; x += kBandThreads)
        band[r * Wp + x] = row[min((long long)x, W - 1)];  // replicate the right edge
    }
  }
  __syncthreads();
  OutT* dst = out + ((img * brows + by) * (long long)bcols) * BB;
  const int total = bcols * BB;
  if constexpr (B % 4 == 0) {
    // four consecutive outputs share (block, row) and are 4-byte aligned in smem
    for (int o4 = threadIdx.x; o4 < total / 4; o4 += kBandThreads) {
      const int o = o4 * 4;
      const int bx = o / BB, q = o % BB, r = q / B, c = q % B;
      const uchar4 p = *reinterpret_cast<const uchar4*>(band + r * Wp + bx * B + c);
      if constexpr (sizeof(OutT) == 4) {
        reinterpret_cast<float4*>(dst)[o4] = make_float4(p.x, p.y, p.z, p.w);
      } else {
        reinterpret_cast<double2*>(dst)[2 * o4] = make_double2(p.x, p.y);
        reinterpret_cast<double2*>(dst)[2 * o4 + 1] = make_double2(p.z, p.w);
      }
    }
  } else {
    for (int o = threadIdx.x; o < total; o += kBandThreads) {
      const int bx = o / BB, q = o % BB, r = q / B, c = q % B;
      dst[o] = (OutT)band[r * Wp + bx * B + c];
    }
  }
}

// Any block side / width: one thread per output element.
template <typename OutT>
__global__ void pixels_to_blocks_generic(const unsigned char* __restrict__ px, long long H,
                                         long long W, long long B, long long bcols,
                                         long long per_img, long long total, OutT* __restrict__ out) {
  const long long BB = B * B;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long img = e / per_img, rem = e % per_img;
    const long long v = rem / BB, q = rem % BB;
    const long long y = min((v / bcols) * B + q / B, H - 1);
    const long long x = min((v % bcols) * B + q % B, W - 1);
    out[e] = (OutT)px[img * H * W + y * W + x];
  }
}

// ---------------------------------------------------------------------------
// block vectors (or codebook indices) -> pixels
// ---------------------------------------------------------------------------

// storage.py:307: np.floor(np.clip(v, 0, 255) + 0.5).astype(np.uint8).
// fmax/fmin return the non-NaN operand, so NaN -> 0 (numpy's x86 cast of NaN).
__device__ __forceinline__ unsigned char quantize(double v) {
  const double c = fmin(fmax(v, 0.0), 255.0);
  return (unsigned char)floor(__dadd_rn(c, 0.5));
}

// Source of a band's values: vectors (vecs != nullptr) or codebook rows
// selected by indices (decode fused with the raster).
template <int B, typename InT>
__global__ void __launch_bounds__(kBandThreads) blocks_to_pixels_band(
    const InT* __restrict__ vecs, const unsigned* __restrict__ idx, const double* __restrict__ cb,
    long long H, long long W, int bcols, int brows, unsigned char* __restrict__ out) {
  extern __shared__ unsigned char band[];  // [B][Wp]
  constexpr int BB = B * B;
  const long long img = blockIdx.y;
  const int by = blockIdx.x;
  const int Wp = bcols * B;
  const long long v0 = (img * brows + by) * (long long)bcols;
  const int total = bcols * BB;
  for (int o = threadIdx.x; o < total; o += kBandThreads) {
    const int bx = o / BB, q = o % BB, r = q / B, c = q % B;
    const double v = vecs ? (double)vecs[v0 * BB + o] : __ldg(cb + (long long)__ldg(idx + v0 + bx) * BB + q);
    band[r * Wp + bx * B + c] = quantize(v);
  }
  __syncthreads();
  unsigned char* dst = out + img * H * W;
  for (int r = 0; r < B; ++r) {
    const long long y = (long long)by * B + r;
    if (y >= H) break;  // crop the bottom padding
    for (int x = threadIdx.x; x < W; x += kBandThreads) dst[y * W + x] = band[r * Wp + x];
  }
}

// decode fused with the raster, B % 4 == 0 and W % 4 == 0: the codebook is
// quantised once (cbq = quantize(cb), K x BB bytes, L1/L2-resident), then one
// thread per 4 horizontally adjacent pixels (same block row, same block):
// one index load (shared by B/4 threads), one 4-byte codebook load, one 4-byte
// coalesced store.  blockIdx.y = image row (img * H + y).
__global__ void quantize_codebook_kernel(const double* __restrict__ cb, long long count,
                                         unsigned char* __restrict__ cbq) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x)
    cbq[e] = quantize(cb[e]);
}

template <int B>
__global__ void __launch_bounds__(256) decode_pixels_vec4(const unsigned* __restrict__ idx,
                                                          const unsigned char* __restrict__ cbq, long long H,
                                                          int W, int bcols, int brows,
                                                          unsigned char* __restrict__ out) {
  constexpr int BB = B * B;
  const long long row = blockIdx.y;  // img * H + y
  const long long img = row / H, y = row - img * H;
  const int x = (blockIdx.x * 256 + threadIdx.x) * 4;
  if (x >= W) return;
  const long long v = (img * brows + y / B) * bcols + x / B;
  const int q = (int)(y % B) * B + x % B;
  const unsigned k = __ldg(idx + v);
  const unsigned p = __ldg(reinterpret_cast<const unsigned*>(cbq + (long long)k * BB + q));
  *reinterpret_cast<unsigned*>(out + row * W + x) = p;
}

// W % 16 == 0: one thread per 16 adjacent pixels of a row (one 16-byte
// store), grid-stride over rows x W/16 so that every thread does several.
template <int B>
__global__ void __launch_bounds__(256) decode_pixels_vec16(const unsigned* __restrict__ idx,
                                                           const unsigned char* __restrict__ cbq, long long H,
                                                           int W, int bcols, int brows, long long units,
                                                           unsigned char* __restrict__ out) {
  constexpr int BB = B * B;
  const int w16 = W >> 4;
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < units;
       u += (long long)gridDim.x * blockDim.x) {
    const long long row = u / w16;  // img * H + y
    const int x0 = (int)(u - row * w16) * 16;
    const long long img = row / H, y = row - img * H;
    const long long vrow = (img * brows + y / B) * bcols;
    const int qrow = (int)(y % B) * B;
    unsigned w[4];
#pragma unroll
    for (int part = 0; part < 4; ++part) {
      const int x = x0 + 4 * part;
      const unsigned k = __ldg(idx + vrow + x / B);
      w[part] = __ldg(reinterpret_cast<const unsigned*>(cbq + (long long)k * BB + qrow + x % B));
    }
    *reinterpret_cast<uint4*>(out + row * W + x0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <typename InT>
__global__ void blocks_to_pixels_generic(const InT* __restrict__ vecs, const unsigned* __restrict__ idx,
                                         const double* __restrict__ cb, long long H, long long W,
                                         long long B, long long bcols, long long brows,
                                         long long total, unsigned char* __restrict__ out) {
  const long long BB = B * B;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long img = e / (H * W), rem = e % (H * W);
    const long long y = rem / W, x = rem % W;
    const long long v = (img * brows + y / B) * bcols + x / B;
    const long long q = (y % B) * B + x % B;
    const double val = vecs ? (double)vecs[v * BB + q] : cb[(long long)idx[v] * BB + q];
    out[e] = quantize(val);
  }
}

// ---------------------------------------------------------------------------
// decode: out[j] = codebook[idx[j]]
// ---------------------------------------------------------------------------

// One thread per 16-byte piece of output (L even), four pieces per loop trip
// (the index and codebook loads of all four are issued before any store, so a
// thread keeps four gathers in flight); streaming stores: the rows are written
// once and never re-read by this kernel.
// PC = L / 2 at compile time (16, 32, 64-dim rows) or 0 (runtime).
template <int PC>
__global__ void __launch_bounds__(256) decode_pairs_kernel(const unsigned* __restrict__ idx, long long n,
                                                           int L, const double* __restrict__ cb, long long K,
                                                           double* __restrict__ out, int* __restrict__ bad) {
  const int P = PC ? PC : L / 2;  // double2 pieces per row
  const long long total = n * P;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const double2* __restrict__ cb2 = reinterpret_cast<const double2*>(cb);
  double2* __restrict__ out2 = reinterpret_cast<double2*>(out);
  bool any_bad = false;
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; e + 3 * stride < total; e += 4 * stride) {
    unsigned k[4];
    long long j[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      j[u] = (e + u * stride) / P;
      k[u] = __ldg(idx + j[u]);
      any_bad |= k[u] >= K;
      k[u] = k[u] < K ? k[u] : 0;  // codec.py:110-113 (never read out of range)
    }
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long eu = e + u * stride;
      v[u] = __ldg(cb2 + (long long)k[u] * P + (eu - j[u] * P));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) __stcs(out2 + e + u * stride, v[u]);
  }
  for (; e < total; e += stride) {
    const long long j = e / P;
    unsigned k = __ldg(idx + j);
    any_bad |= k >= K;
    k = k < K ? k : 0;
    __stcs(out2 + e, __ldg(cb2 + (long long)k * P + (e - j * P)));
  }
  if (any_bad) atomicOr(bad, 1);
}

__global__ void decode_elems_kernel(const unsigned* __restrict__ idx, long long n, int L,
                                    const double* __restrict__ cb, long long K, double* __restrict__ out,
                                    int* __restrict__ bad) {
  const long long total = n * L;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / L;
    unsigned k = __ldg(idx + j);
    if (k >= K) {
      atomicOr(bad, 1);
      k = 0;
    }
    out[e] = __ldg(cb + (long long)k * L + (e - j * L));
  }
}

__global__ void index_check_kernel(const unsigned* __restrict__ idx, long long n, long long K,
                                   int* __restrict__ bad) {
  bool any = false;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x)
    any |= __ldg(idx + j) >= K;
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// ---------------------------------------------------------------------------
// reconstruction distortion: per-row pair_distance + sums
// ---------------------------------------------------------------------------

template <int DIM>
__global__ void __launch_bounds__(256) pair_rows_kernel(const double* __restrict__ a,
                                                        const double* __restrict__ b, long long n,
                                                        int dim, int metric, double* __restrict__ d) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    double v = winner_dist<double, DIM>(a + j * (DIM ? DIM : dim), b + j * (DIM ? DIM : dim), dim);
    if (metric == kEuclidean) v = sqrt(v);  // IEEE sqrt, as math.sqrt
    d[j] = v;
  }
}

// Per-tile fixed-tree partials (kTdTile rows per tile), the same tree as the
// training loop's distortion (td_tiles_kernel).
__global__ void __launch_bounds__(256) tile_sums_kernel(const double* __restrict__ v, long long n,
                                                        double* __restrict__ tiles) {
  __shared__ double red[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long t = blockIdx.x;
  double s = 0.0;
#pragma unroll
  for (int r = 0; r < kTdTile / 256; ++r) {
    const long long row = t * kTdTile + (long long)r * 256 + tid;
    s = __dadd_rn(s, row < n ? v[row] : 0.0);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (tid == 0) {
    double acc = 0.0;
    for (int w = 0; w < 8; ++w) acc = __dadd_rn(acc, red[w]);
    tiles[t] = acc;
  }
}

__global__ void inorder_kernel(const double* v, long long n, double* out) {
  double s = 0.0;
  for (long long i = 0; i < n; ++i) s = __dadd_rn(s, v[i]);
  *out = s;
}

// core._split_rows (core.py:277-281): rows 2i = c + delta, 2i+1 = c - delta,
// each component rounded once (the device loop's apply_kernel does the same)
__global__ void split_rows_kernel(const double* __restrict__ cb, long long count, int dim, double delta,
                                  double* __restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / dim, l = e - i * dim;
    const double c = cb[e];
    out[(2 * i) * dim + l] = __dadd_rn(c, delta);
    out[(2 * i + 1) * dim + l] = __dsub_rn(c, delta);
  }
}

int grid_for(long long work, int sms) {
  const long long g = (work + 255) / 256;
  return (int)std::max<long long>(1, std::min<long long>(g, (long long)sms * 8));
}

int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <typename OutT>
cudaError_t launch_p2b(const unsigned char* px, long long images, long long H, long long W, int B,
                       OutT* out, cudaStream_t s) {
  const long long bcols = (W + B - 1) / B, brows = (H + B - 1) / B;
  const long long Wp = bcols * B;
  const size_t smem = (size_t)(B * Wp);
  const bool band = smem <= (size_t)kBandSmem && brows <= INT_MAX && images <= 65535 &&
                    (B == 2 || B == 4 || B == 8 || B == 16);
  if (band) {
    dim3 grid((unsigned)brows, (unsigned)images);
    switch (B) {
      case 2: pixels_to_blocks_band<2, OutT><<<grid, kBandThreads, smem, s>>>(px, H, W, (int)bcols, (int)brows, out); break;
      case 4: pixels_to_blocks_band<4, OutT><<<grid, kBandThreads, smem, s>>>(px, H, W, (int)bcols, (int)brows, out); break;
      case 8: pixels_to_blocks_band<8, OutT><<<grid, kBandThreads, smem, s>>>(px, H, W, (int)bcols, (int)brows, out); break;
      default: pixels_to_blocks_band<16, OutT><<<grid, kBandThreads, smem, s>>>(px, H, W, (int)bcols, (int)brows, out); break;
    }
  } else {
    const long long per_img = bcols * brows * (long long)B * B;
    const long long total = per_img * images;
    pixels_to_blocks_generic<OutT><<<grid_for(total, device_sms()), 256, 0, s>>>(px, H, W, B, bcols, per_img,
                                                                                total, out);
  }
  return cudaGetLastError();
}

template <typename InT>
cudaError_t launch_b2p(const InT* vecs, const unsigned* idx, const double* cb, long long images,
                       long long H, long long W, int B, unsigned char* out, cudaStream_t s) {
  const long long bcols = (W + B - 1) / B, brows = (H + B - 1) / B;
  const long long Wp = bcols * B;
  const size_t smem = (size_t)(B * Wp);
  const bool band = smem <= (size_t)kBandSmem && brows <= INT_MAX && images <= 65535 &&
                    (B == 2 || B == 4 || B == 8 || B == 16);
  if (band) {
    dim3 grid((unsigned)brows, (unsigned)images);
    switch (B) {
      case 2: blocks_to_pixels_band<2, InT><<<grid, kBandThreads, smem, s>>>(vecs, idx, cb, H, W, (int)bcols, (int)brows, out); break;
      case 4: blocks_to_pixels_band<4, InT><<<grid, kBandThreads, smem, s>>>(vecs, idx, cb, H, W, (int)bcols, (int)brows, out); break;
      case 8: blocks_to_pixels_band<8, InT><<<grid, kBandThreads, smem, s>>>(vecs, idx, cb, H, W, (int)bcols, (int)brows, out); break;
      default: blocks_to_pixels_band<16, InT><<<grid, kBandThreads, smem, s>>>(vecs, idx, cb, H, W, (int)bcols, (int)brows, out); break;
    }
  } else {
    const long long total = images * H * W;
    blocks_to_pixels_generic<InT><<<grid_for(total, device_sms()), 256, 0, s>>>(vecs, idx, cb, H, W, B, bcols,
                                                                               brows, total, out);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_pixels_to_blocks_f32(const unsigned char* px, long long images, long long H, long long W,
                                        int block, float* out, cudaStream_t s) {
  return launch_p2b<float>(px, images, H, W, block, out, s);
}

cudaError_t launch_pixels_to_blocks_f64(const unsigned char* px, long long images, long long H, long long W,
                                        int block, double* out, cudaStream_t s) {
  return launch_p2b<double>(px, images, H, W, block, out, s);
}

cudaError_t launch_blocks_to_pixels(const double* vecs, const unsigned* idx, const double* cb, long long images,
                                    long long H, long long W, int block, unsigned char* out, cudaStream_t s) {
  return launch_b2p<double>(vecs, idx, cb, images, H, W, block, out, s);
}

cudaError_t launch_decode_pixels(const unsigned* idx, const double* cb, long long K, long long images,
                                 long long H, long long W, int block, unsigned char* cbq, unsigned char* out,
                                 cudaStream_t s) {
  const long long rows = images * H;
  const bool vec4 = (block == 4 || block == 8 || block == 16) && (W % 4) == 0 &&
                    (rows <= 65535 || W % 16 == 0) && W <= INT_MAX;
  if (!vec4) return launch_b2p<double>(nullptr, idx, cb, images, H, W, block, out, s);
  const long long bb = (long long)block * block;
  quantize_codebook_kernel<<<grid_for(K * bb, device_sms()), 256, 0, s>>>(cb, K * bb, cbq);
  const int bcols = (int)((W + block - 1) / block), brows = (int)((H + block - 1) / block);
  if (W % 16 == 0) {
    const long long units = rows * (W / 16);
    const int g = grid_for(units, device_sms());
    switch (block) {
      case 4: decode_pixels_vec16<4><<<g, 256, 0, s>>>(idx, cbq, H, (int)W, bcols, brows, units, out); break;
      case 8: decode_pixels_vec16<8><<<g, 256, 0, s>>>(idx, cbq, H, (int)W, bcols, brows, units, out); break;
      default: decode_pixels_vec16<16><<<g, 256, 0, s>>>(idx, cbq, H, (int)W, bcols, brows, units, out); break;
    }
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((W / 4 + 255) / 256), (unsigned)rows);
  switch (block) {
    case 4: decode_pixels_vec4<4><<<grid, 256, 0, s>>>(idx, cbq, H, (int)W, bcols, brows, out); break;
    case 8: decode_pixels_vec4<8><<<grid, 256, 0, s>>>(idx, cbq, H, (int)W, bcols, brows, out); break;
    default: decode_pixels_vec4<16><<<grid, 256, 0, s>>>(idx, cbq, H, (int)W, bcols, brows, out); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_decode(const unsigned* idx, long long n, int L, const double* cb, long long K, double* out,
                          int* bad, cudaStream_t s) {
  const int sms = device_sms();
  const int g = grid_for(n * (L / 2), sms);
  if (L == 16)
    decode_pairs_kernel<8><<<g, 256, 0, s>>>(idx, n, L, cb, K, out, bad);
  else if (L == 64)
    decode_pairs_kernel<32><<<g, 256, 0, s>>>(idx, n, L, cb, K, out, bad);
  else if (L % 2 == 0)
    decode_pairs_kernel<0><<<g, 256, 0, s>>>(idx, n, L, cb, K, out, bad);
  else
    decode_elems_kernel<<<grid_for(n * L, sms), 256, 0, s>>>(idx, n, L, cb, K, out, bad);
  return cudaGetLastError();
}

cudaError_t launch_split_rows(const double* cb, long long size, int dim, double delta, double* out,
                              cudaStream_t s) {
  const long long count = size * dim;
  split_rows_kernel<<<grid_for(count, device_sms()), 256, 0, s>>>(cb, count, dim, delta, out);
  return cudaGetLastError();
}

cudaError_t launch_index_check(const unsigned* idx, long long n, long long K, int* bad, cudaStream_t s) {
  index_check_kernel<<<grid_for(n, device_sms()), 256, 0, s>>>(idx, n, K, bad);
  return cudaGetLastError();
}

// Per-row pair distances into d[n]; total = in-order sum when n <= inorder_max,
// else per-tile fixed tree + in-order over tiles (tiles[ceil(n / kTdTile)]).
cudaError_t launch_pair_rows(const double* a, const double* b, long long n, int dim, int metric, double* d,
                             cudaStream_t s) {
  const int g = grid_for(n, device_sms());
  if (dim == 16)
    pair_rows_kernel<16><<<g, 256, 0, s>>>(a, b, n, dim, metric, d);
  else if (dim == 64)
    pair_rows_kernel<64><<<g, 256, 0, s>>>(a, b, n, dim, metric, d);
  else
    pair_rows_kernel<0><<<g, 256, 0, s>>>(a, b, n, dim, metric, d);
  return cudaGetLastError();
}

cudaError_t launch_distortion_sum(const double* d, long long n, bool inorder, double* tiles, double* out,
                                  cudaStream_t s) {
  if (inorder) {
    inorder_kernel<<<1, 1, 0, s>>>(d, n, out);
  } else {
    const long long nt = (n + kTdTile - 1) / kTdTile;
    tile_sums_kernel<<<(unsigned)nt, 256, 0, s>>>(d, n, tiles);
    inorder_kernel<<<1, 1, 0, s>>>(tiles, nt, out);
  }
  return cudaGetLastError();
}

}  // namespace vqb
