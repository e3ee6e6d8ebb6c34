// FP32/FP64 pipe microbenchmarks: the measured denominator for the roofline
// of the distance pass (BASELINE.md section 4 asks for a measured FFMA peak
// beside the nominal SMs x 128 x 2 x f_clk).  Each kernel runs independent
// dependency chains so the pipe, not latency, is the limit.
#include <cstdint>
#include <cuda_runtime.h>

#include "vqb200_internal.h"

namespace vqb {

template <int CHAINS>
__global__ void __launch_bounds__(256) ffma_kernel(float* out, int iters, float a, float b) {
  float acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-7f + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] = fmaf(acc[c], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 123.456f) out[0] = s;
}

// packed f32x2 FMA (sm_100+: FFMA2)
template <int CHAINS>
__global__ void __launch_bounds__(256) ffma2_kernel(float* out, int iters, float a, float b) {
  unsigned long long acc[CHAINS];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long ab = *reinterpret_cast<unsigned long long*>(&av);
  unsigned long long bb = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    float2 v = make_float2(threadIdx.x * 1e-7f + c, c * 0.5f);
    acc[c] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[c]) : "l"(ab), "l"(bb));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    float2 v = *reinterpret_cast<float2*>(&acc[c]);
    s += v.x + v.y;
  }
  if (s == 123.456f) out[0] = s;
}

// 16 FFMA + top-2 bookkeeping (FSETP, SEL, 3 FMNMX) per "eval": the
// expanded-form distance inner loop shape, to measure ALU co-issue.
template <int CHAINS>
__global__ void __launch_bounds__(256) mix_kernel(float* out, int iters, float a, float b) {
  float acc[CHAINS], m1[CHAINS], m2[CHAINS];
  int i1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    acc[c] = threadIdx.x * 1e-7f + c;
    m1[c] = 3e38f;
    m2[c] = 3e38f;
    i1[c] = 0;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      float v = acc[c];
#pragma unroll
      for (int k = 0; k < 16; ++k) v = fmaf(v, a, b);
      acc[c] = v;
      m2[c] = fminf(m2[c], fmaxf(m1[c], v));
      bool p = v < m1[c];
      m1[c] = fminf(m1[c], v);
      i1[c] = p ? it : i1[c];
    }
  }
  float s = 0.f;
  int si = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    s += m1[c] + m2[c];
    si += i1[c];
  }
  if (s == 123.456f || si == -7) out[0] = s + si;
}

template <int CHAINS>
__global__ void __launch_bounds__(256) dadd_kernel(double* out, int iters, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-7 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] = __dadd_rn(acc[c], b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 123.456) out[0] = s;
}

// 3 vector-register operands (no uniform / constant / immediate source)
template <int CHAINS>
__global__ void __launch_bounds__(256) ffma3r_kernel(float* out, const float* in, int iters) {
  float acc[CHAINS], xa[CHAINS], xb[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    acc[c] = in[(threadIdx.x + c) & 255];
    xa[c] = in[(threadIdx.x * 3 + c) & 255];
    xb[c] = in[(threadIdx.x * 5 + c) & 255];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] = fmaf(xa[c], acc[c], xb[c]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 123.456f) out[0] = s;
}

// distance inner loop, codebook in __constant__ (ULDC -> uniform registers)
__constant__ float c_mb_cb[512 * 17];

template <int R>
__global__ void __launch_bounds__(256) dist_const_kernel(float* out, const float* in, int K, int reps) {
  float y[R][16];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int l = 0; l < 16; ++l) y[r][l] = in[(threadIdx.x * 7 + r * 16 + l) & 255];
  float m1[R], m2[R];
  int i1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { m1[r] = INFINITY; m2[r] = INFINITY; i1[r] = 0; }
  for (int rep = 0; rep < reps; ++rep) {
    for (int j = 0; j < K; ++j) {
      float v[R];
      const float nj = c_mb_cb[j * 17 + 16];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = nj;
#pragma unroll
      for (int l = 0; l < 16; ++l) {
        const float w = c_mb_cb[j * 17 + l];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = fmaf(w, y[r][l], v[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float n2 = fminf(m2[r], fmaxf(m1[r], v[r]));
        const bool p = v[r] < m1[r];
        m1[r] = fminf(m1[r], v[r]);
        i1[r] = p ? j : i1[r];
        m2[r] = n2;
      }
    }
  }
  float s = 0.f;
  int si = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) { s += m1[r] + m2[r]; si += i1[r]; }
  if (s == 123.456f || si == -7) out[0] = s + si;
}


// FFMA2 and scalar FFMA interleaved (independent chains): does the scalar
// FFMA co-issue on the fmalite half while FFMA2 occupies fmaheavy?
template <int CHAINS>
__global__ void __launch_bounds__(256) ffma2_mix_kernel(float* out, int iters, float a, float b) {
  unsigned long long acc[CHAINS];
  float sc[CHAINS];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long ab = *reinterpret_cast<unsigned long long*>(&av);
  unsigned long long bb = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    float2 v = make_float2(threadIdx.x * 1e-7f + c, c * 0.5f);
    acc[c] = *reinterpret_cast<unsigned long long*>(&v);
    sc[c] = threadIdx.x * 3e-7f + c;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) {
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[c]) : "l"(ab), "l"(bb));
        sc[c] = fmaf(sc[c], a, b);
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    float2 v = *reinterpret_cast<float2*>(&acc[c]);
    s += v.x + v.y + sc[c];
  }
  if (s == 123.456f) out[0] = s;
}

// ALU-pipe rate: FMNMX chains (top-2 bookkeeping is FMNMX/FSETP/SEL)
template <int CHAINS>
__global__ void __launch_bounds__(256) fmnmx_kernel(float* out, int iters, float a) {
  float acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-7f + c;
  for (int it = 0; it < iters; ++it) {
    const float t = a + it;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] = fminf(acc[c], (k & 1) ? -t : t);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 123.456f) out[0] = s;
}


// ALU-pipe probes for the top-2 epilogue: FMNMX (two register operands),
// integer VIMNMX, and the two interleaved (do they share one pipe?)
template <int CHAINS, int MODE>
__global__ void __launch_bounds__(256) minmax_kernel(float* out, const float* in, int iters) {
  float fa[CHAINS], fb[CHAINS];
  int ia[CHAINS], ib[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    fa[c] = in[(threadIdx.x + c) & 255];
    fb[c] = in[(threadIdx.x * 3 + c) & 255];
    ia[c] = __float_as_int(fa[c]) ^ c;
    ib[c] = __float_as_int(fb[c]) + c;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) {
        if (MODE == 0 || MODE == 2) {
          asm volatile("min.f32 %0, %0, %1;" : "+f"(fa[c]) : "f"(fb[c]));
          asm volatile("max.f32 %0, %0, %1;" : "+f"(fb[c]) : "f"(fa[c]));
        }
        if (MODE == 1 || MODE == 2) {
          asm volatile("min.s32 %0, %0, %1;" : "+r"(ia[c]) : "r"(ib[c]));
          asm volatile("max.s32 %0, %0, %1;" : "+r"(ib[c]) : "r"(ia[c]));
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += fa[c] + fb[c] + (float)(ia[c] + ib[c]);
  if (s == 123.456f) out[0] = s;
}


// 3-input FMNMX3 with three register operands (the single-read top-2 epilogue
// is ~80 % FMNMX3): MODE 0 = min3 / max3 chains, MODE 1 = the epilogue's mix
// per 32 values (16 class chains + 2 block minima + 2 top-2 folds)
template <int MODE>
__global__ void __launch_bounds__(256) fmnmx3_kernel(float* out, const float* in, int iters) {
  float fa[8], fb[8], fc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    fa[c] = in[(threadIdx.x + c) & 255];
    fb[c] = in[(threadIdx.x * 3 + c) & 255];
    fc[c] = in[(threadIdx.x * 5 + c) & 255];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        fa[c] = fminf(fminf(fb[c], fc[c]), fa[c]);
        fb[c] = fmaxf(fmaxf(fc[c], fa[c]), fb[c]);
        if (MODE == 1) fc[c] = fminf(fc[c], fmaxf(fa[c], fb[(c + 1) & 7]));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += fa[c] + fb[c] + fc[c];
  if (s == 123.456f) out[0] = s;
}

// shared-memory atomics for the cell tables: non-returning adds (RED) vs
// returning adds whose result feeds a dependent add (the 64-bit carry idiom)
template <int MODE>
__global__ void __launch_bounds__(512) smem_atomic_kernel(float* out, int iters) {
  __shared__ unsigned tab[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  unsigned h = threadIdx.x * 2654435761u + blockIdx.x;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      h = h * 1664525u + 1013904223u;
      const unsigned a = (h >> 8) & 8191u;
      if (MODE == 0) {
        atomicAdd(&tab[a], 1u);
      } else {
        const unsigned old = atomicAdd(&tab[a], 3u);
        if (old + 3u < old) atomicAdd(&tab[(a + 1) & 8191u], 1u);
        acc += old;
      }
    }
  }
  __syncthreads();
  if (tab[threadIdx.x] == 0xdeadbeef || acc == 7u) out[0] = 1.f;
}


// HBM read patterns of the epilogue passes over X [N][16] f32 (64 MiB):
// MODE 0: one row per thread (4 x float4 per lane, rows 64 B apart),
// MODE 1: fully coalesced float4 stream (consecutive lanes, consecutive 16 B)
template <int MODE>
__global__ void __launch_bounds__(256) xread_kernel(const float4* __restrict__ x, long long rows, float* out) {
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (MODE == 0) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += stride) {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const float4 q = __ldg(x + r * 4 + v);
        acc += q.x + q.y + q.z + q.w;
      }
    }
  } else {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows * 4; i += stride) {
      const float4 q = __ldg(x + i);
      acc += q.x + q.y + q.z + q.w;
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

}  // namespace vqb

using namespace vqb;

// Returns achieved lane-ops/s (FMA counted once) for pipe `which`:
// 0 = FFMA, 1 = FFMA2 (2 lane-ops per instruction), 2 = 16xFFMA + top-2 mix
// (counts the 16 FFMA only), 3 = DADD, 4 = 3-register FFMA, 5 = evals/s of a
// constant-memory-codebook distance loop, 6 = FFMA2 + FFMA interleaved (FMA
// lane-ops), 7 = FMNMX (ALU pipe).  `seconds` gets the kernel time.
// L2 (global) 64-bit atomics into a K x 17 int64 cell table (the fused
// cell-sum candidate): each thread plays one row, picks a pseudo-random cell
// and adds 17 words (16 dims + count) -- MODE 0 non-returning red.add.u64,
// MODE 1 the same words from 32 lanes of one warp coalesced per dim (lane =
// row, consecutive dims per instruction).
template <int MODE>
__global__ void __launch_bounds__(256) l2_red_kernel(unsigned long long* tab, int cells, int iters) {
  unsigned h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    const unsigned cell = (h >> 8) % (unsigned)cells;
    unsigned long long* w = tab + (unsigned long long)cell * 17;
#pragma unroll
    for (int d = 0; d < 17; ++d) atomicAdd(w + d, (unsigned long long)(h & 0xffff) + d);
  }
}

extern "C" int vqb_pipe_microbench(int which, int blocks_per_sm, int iters, double* ops_per_s,
                                   double* seconds) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256;
  const int blocks = sms * blocks_per_sm;
  void* buf = nullptr;
  void* inbuf = nullptr;
  if (cudaMalloc(&buf, 64) != cudaSuccess) return 4;
  if (cudaMalloc(&inbuf, 1024) != cudaSuccess) return 4;
  cudaMemset(inbuf, 0, 1024);
  {
    static float hcb[512 * 17];
    for (int i = 0; i < 512 * 17; ++i) hcb[i] = (float)((i * 37) % 101) * 0.01f;
    cudaMemcpyToSymbol(c_mb_cb, hcb, sizeof(hcb));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double lane_ops = 0;
  for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
    cudaEventRecord(e0);
    switch (which) {
      case 0:
        ffma_kernel<8><<<blocks, threads>>>((float*)buf, iters, 0.999f, 1e-3f);
        lane_ops = 1.0 * blocks * threads * iters * 16 * 8;
        break;
      case 1:
        ffma2_kernel<8><<<blocks, threads>>>((float*)buf, iters, 0.999f, 1e-3f);
        lane_ops = 2.0 * blocks * threads * iters * 16 * 8;
        break;
      case 2:
        mix_kernel<8><<<blocks, threads>>>((float*)buf, iters, 0.999f, 1e-3f);
        lane_ops = 1.0 * blocks * threads * iters * 16 * 8;
        break;
      case 3:
        dadd_kernel<8><<<blocks, threads>>>((double*)buf, iters, 1e-3);
        lane_ops = 1.0 * blocks * threads * iters * 16 * 8;
        break;
      case 4:
        ffma3r_kernel<8><<<blocks, threads>>>((float*)buf, (const float*)inbuf, iters);
        lane_ops = 1.0 * blocks * threads * iters * 16 * 8;
        break;
      case 6:
        ffma2_mix_kernel<8><<<blocks, threads>>>((float*)buf, iters, 0.999f, 1e-3f);
        lane_ops = 3.0 * blocks * threads * iters * 16 * 8;
        break;
      case 7:
        fmnmx_kernel<8><<<blocks, threads>>>((float*)buf, iters, 0.5f);
        lane_ops = 1.0 * blocks * threads * iters * 16 * 8;
        break;
      case 8:
      case 9:
      case 10: {
        const int mode = which - 8;
        if (mode == 0) minmax_kernel<8, 0><<<blocks, threads>>>((float*)buf, (const float*)inbuf, iters);
        if (mode == 1) minmax_kernel<8, 1><<<blocks, threads>>>((float*)buf, (const float*)inbuf, iters);
        if (mode == 2) minmax_kernel<8, 2><<<blocks, threads>>>((float*)buf, (const float*)inbuf, iters);
        lane_ops = (mode == 2 ? 4.0 : 2.0) * blocks * threads * iters * 8 * 8;
        break;
      }
      case 17:
      case 18:
        if (which == 17) fmnmx3_kernel<0><<<blocks, threads>>>((float*)buf, (const float*)inbuf, iters);
        else fmnmx3_kernel<1><<<blocks, threads>>>((float*)buf, (const float*)inbuf, iters);
        lane_ops = (which == 17 ? 2.0 : 4.0) * blocks * threads * iters * 4 * 8;  // instructions x lanes
        break;
      case 11:
      case 12:
        if (which == 11) smem_atomic_kernel<0><<<sms, 512>>>((float*)buf, iters);
        else smem_atomic_kernel<1><<<sms, 512>>>((float*)buf, iters);
        lane_ops = 1.0 * sms * 512 * iters * 16;
        break;
      case 15:
      case 16: {
        static unsigned long long* tab = nullptr;
        const int cells = which == 15 ? 1024 : 4096;
        if (!tab) {
          cudaMalloc(&tab, 4096ull * 17 * 8);
          cudaMemset(tab, 0, 4096ull * 17 * 8);
        }
        const int it = iters / 20 + 1;
        l2_red_kernel<0><<<sms * 8, 256>>>(tab, cells, it);
        lane_ops = 17.0 * sms * 8 * 256 * it;
        break;
      }
      case 13:
      case 14: {
        static float4* xb = nullptr;
        const long long rows = 1LL << 20;
        if (!xb) {
          cudaMalloc(&xb, rows * 64);
          cudaMemset(xb, 0, rows * 64);
        }
        if (which == 13) xread_kernel<0><<<sms * 8, 256>>>(xb, rows, (float*)buf);
        else xread_kernel<1><<<sms * 8, 256>>>(xb, rows, (float*)buf);
        lane_ops = (double)rows * 64;  // bytes
        break;
      }
      default:  // 5: evals/s of the constant-codebook distance loop (K=512, R=4)
        dist_const_kernel<4><<<blocks, threads>>>((float*)buf, (const float*)inbuf, 512, iters / 100 + 1);
        lane_ops = 1.0 * blocks * threads * 4 * 512 * (iters / 100 + 1);
        break;
    }
    cudaEventRecord(e1);
  }
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(inbuf);
  if (err != cudaSuccess) return 4;
  *seconds = ms * 1e-3;
  *ops_per_s = lane_ops / (ms * 1e-3);
  return 0;
}
