// The reference's FP64 distance arithmetic on the device (_kernels.py:25-34):
// for c ascending, diff = x - c; d = d + diff * diff, every operation rounded
// separately (the _rn intrinsics forbid FMA contraction).
#pragma once
#include <cuda_runtime.h>

namespace vqb {

__device__ __forceinline__ double load_x(const float* x, long long i) { return (double)x[i]; }
__device__ __forceinline__ double load_x(const double* x, long long i) { return x[i]; }

// Squared distance in the reference's arithmetic (_kernels.py:25-29): for c
// ascending, diff = x - c; d = d + diff*diff, every op rounded separately
// (the _rn intrinsics forbid FMA contraction).
template <typename XT>
__device__ __forceinline__ double ref_dist(const XT* x, const double* c, int dim) {
  double d = 0.0;
  for (int l = 0; l < dim; ++l) {
    double diff = __dsub_rn(load_x(x, l), c[l]);
    d = __dadd_rn(d, __dmul_rn(diff, diff));
  }
  return d;
}

// ref_dist with vectorised loads for a compile-time row length (DIM = 0:
// runtime length).  Float rows widen exactly (core.py:47-60).
template <typename XT, int DIM>
__device__ __forceinline__ double winner_dist(const XT* __restrict__ x, const double* __restrict__ c,
                                              int dim) {
  double d = 0.0;
  if constexpr (DIM > 0) {
#pragma unroll
    for (int c0 = 0; c0 < DIM; c0 += 16) {
      double xr[16], cr[16];
      if constexpr (sizeof(XT) == 4) {
        const float4* x4 = reinterpret_cast<const float4*>(x + c0);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const float4 q = __ldg(x4 + v);
          xr[4 * v] = q.x;
          xr[4 * v + 1] = q.y;
          xr[4 * v + 2] = q.z;
          xr[4 * v + 3] = q.w;
        }
      } else {
        const double2* x2 = reinterpret_cast<const double2*>(x + c0);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const double2 q = __ldg(x2 + v);
          xr[2 * v] = q.x;
          xr[2 * v + 1] = q.y;
        }
      }
      const double2* c2 = reinterpret_cast<const double2*>(c + c0);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const double2 q = __ldg(c2 + v);
        cr[2 * v] = q.x;
        cr[2 * v + 1] = q.y;
      }
#pragma unroll
      for (int l = 0; l < 16; ++l) {
        const double diff = __dsub_rn(xr[l], cr[l]);
        d = __dadd_rn(d, __dmul_rn(diff, diff));
      }
    }
  } else {
    d = ref_dist(x, c, dim);
  }
  return d;
}

}  // namespace vqb
