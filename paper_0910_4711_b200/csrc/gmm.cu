// Device-side Gaussian-mixture training rows (the
// generators on the GPU, so cfg2/cfg4/cfg5-sized inputs never cross PCIe).
//
// Counter-based: row r draws from Philox4x32-10 with counter (r_lo, r_hi,
// call, 0) and key (seed_lo, seed_hi) -- call 0 picks the component, calls
// 1.. give the uniforms of the Box-Muller pairs -- so every row is
// independent of the grid and of every other row.  The component parameters
// (means, sigmas, cumulative weights; a few KB) come from the host.
//
// The arithmetic uses only IEEE add / sub / mul / div / sqrt on doubles
// (logarithm and sine / cosine by fixed series), and this file is compiled
// with -fmad=false, so a host restatement with the same operation order and
// no FMA contraction (oracle/oracle.py gmm_rows) reproduces every float bit.
#include <cstdint>

#include "vqb200_internal.h"

namespace vqb {

struct Philox {
  uint32_t v[4];
};

__device__ __forceinline__ Philox philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                           uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c0 = n0;
    c1 = (uint32_t)p1;
    c2 = n2;
    c3 = (uint32_t)p0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  Philox o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}

// 1 / k! (k < 22) and 1 / (2k + 1) (k < 14) as IEEE quotients of exact
// operands: the host restatement divides at run time and gets the same bits
__constant__ double kInvFact[22] = {1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333, 0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06, 2.755731922398589e-07, 2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10, 1.1470745597729725e-11, 7.647163731819816e-13, 4.779477332387385e-14, 2.8114572543455206e-15, 1.5619206968586225e-16, 8.22063524662433e-18, 4.110317623312165e-19, 1.9572941063391263e-20};
__constant__ double kInvOdd[14] = {1.0, 0.3333333333333333, 0.2, 0.14285714285714285, 0.1111111111111111, 0.09090909090909091, 0.07692307692307693, 0.06666666666666667, 0.058823529411764705, 0.05263157894736842, 0.047619047619047616, 0.043478260869565216, 0.04, 0.037037037037037035};

// uniform in (0, 1): (x + 1/2) 2^-32
__device__ __forceinline__ double unit(uint32_t x) { return ((double)x + 0.5) * 2.3283064365386963e-10; }

// natural log of u in (0, 1): u = m 2^e with m in [1, 2), log m = 2 atanh(s),
// s = (m - 1) / (m + 1), by 14 terms of the odd series
__device__ __forceinline__ double gmm_log(double u) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(u);
  const int e = (int)((b >> 52) & 0x7ff) - 1023;
  const double m = __longlong_as_double((long long)((b & 0xfffffffffffffull) | 0x3ff0000000000000ull));
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  double t = kInvOdd[13];
#pragma unroll
  for (int k = 12; k >= 0; --k) t = kInvOdd[k] + s2 * t;
  return (double)e * 0.6931471805599453 + 2.0 * s * t;
}

// sin and cos of 2 pi u, u in (0, 1): quadrant q = floor(4 u), angle
// f pi / 2 with f = 4 u - q in [0, 1), Taylor series to x^21 / x^20
__device__ __forceinline__ void gmm_sincos(double u, double& sn, double& cs) {
  const double t = u * 4.0;
  const int q = (int)t;
  const double x = (t - (double)q) * 1.5707963267948966;
  const double x2 = x * x;
  double ps = kInvFact[21];
  double pc = kInvFact[20];
#pragma unroll
  for (int k = 9; k >= 0; --k) {
    ps = kInvFact[2 * k + 1] - x2 * ps;
    pc = kInvFact[2 * k] - x2 * pc;
  }
  const double s0 = x * ps, c0 = pc;
  switch (q & 3) {
    case 0: sn = s0; cs = c0; break;
    case 1: sn = c0; cs = -s0; break;
    case 2: sn = -s0; cs = -c0; break;
    default: sn = -c0; cs = s0; break;
  }
}

// One row per thread: component c (uniform, or the first cumulative weight
// above a uniform), then x_l = mean_c,l + sigma_c z_l with z from Box-Muller
// pairs, rounded to float32.
__global__ void gmm_rows_kernel(const float* __restrict__ means, const float* __restrict__ sigmas,
                                const double* __restrict__ cw, long long comps, long long rows, int dim,
                                long long row0, uint32_t k0, uint32_t k1, float* __restrict__ out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    const long long g = row0 + r;  // global row: shards draw their own slice
    const uint32_t rl = (uint32_t)g, rh = (uint32_t)(g >> 32);
    const double uc = unit(philox10(rl, rh, 0u, 0u, k0, k1).v[0]);
    long long c;
    if (cw) {  // first i with uc < cw[i] (binary search; cw[comps - 1] == 1)
      long long lo = 0, hi = comps - 1;
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (uc < cw[mid]) hi = mid; else lo = mid + 1;
      }
      c = lo;
    } else {
      c = (long long)(uc * (double)comps);
      if (c >= comps) c = comps - 1;
    }
    const double sg = (double)sigmas[c];
    const float* mu = means + c * dim;
    float* o = out + r * dim;
    for (int l0 = 0; l0 < dim; l0 += 4) {
      const Philox ph = philox10(rl, rh, (uint32_t)(1 + l0 / 4), 0u, k0, k1);
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const double u1 = unit(ph.v[2 * p]), u2 = unit(ph.v[2 * p + 1]);
        const double rad = sqrt(-2.0 * gmm_log(u1));
        double sn, cs;
        gmm_sincos(u2, sn, cs);
        const int l = l0 + 2 * p;
        if (l < dim) o[l] = (float)((double)mu[l] + sg * (rad * cs));
        if (l + 1 < dim) o[l + 1] = (float)((double)mu[l + 1] + sg * (rad * sn));
      }
    }
  }
}

cudaError_t launch_gmm_rows(const float* means, const float* sigmas, const double* cw, long long comps,
                            long long rows, int dim, long long row0, unsigned long long seed, float* out, int sms,
                            cudaStream_t s) {
  gmm_rows_kernel<<<sms * 8, 256, 0, s>>>(means, sigmas, cw, comps, rows, dim, row0, (uint32_t)seed,
                                          (uint32_t)(seed >> 32), out);
  return cudaGetLastError();
}

}  // namespace vqb
