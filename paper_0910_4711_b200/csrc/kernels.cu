// sm_100a kernels for the LBG hot path (arxiv/paper_0910_4711 reference:
// pkg/src/vqkit/_kernels.py, core.py, parallel.py).
//
//   prep_codebook     FP64 master codebook -> centred FP32 staging (w=-2c~, ||c~||^2)
//   assign_fast<L>    nearest-codevector candidate pass: FP32 FFMA expanded form,
//                     codebook tiles staged in smem by cp.async.bulk (TMA bulk
//                     copies) + mbarrier, rows in registers, top-2 per row,
//                     rigorous error band -> rows it cannot certify go to
//   exact_rows        FP64 scan in the reference's exact arithmetic
//                     (_kernels.py:22-32: dsub, dmul, dadd, ascending c, strict <)
//   epilogue          exact FP64 winner distance, deterministic distortion tile
//                     partials, int64 fixed-point cell sums + counts (order-free,
//                     hence deterministic and G-invariant)
//   ordered_update    reference-order FP64 cell sums (update_rows, _kernels.py:39-66),
//                     used for float64 inputs where bit-identity needs the order
//   finalize          one block: distortion, convergence test (core.py:342-356),
//                     centroid update / empty cells (_kernels.py:59-66), split
//                     (core.py:277-281), level/guard logic (core.py:384-415), history
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "ptx.h"
#include "refarith.cuh"
#include "vqb200_internal.h"

namespace vqb {

// packed f32x2 (sm_100 FFMA2): two rows' accumulators in one 64-bit register
// pair; the codebook value is a scalar broadcast operand (R.F32 in SASS).
__device__ __forceinline__ unsigned long long pack2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// the row's exact distance to its winner (reference arithmetic; sqrt under
// euclidean, _kernels.py:33-34) -- every assignment path stores it, so the
// distortion pass only reads dists
__device__ __forceinline__ void store_dist(const KernelArgs& a, long long row, double d) {
  if (a.dists) a.dists[row] = a.st->metric == kEuclidean ? sqrt(d) : d;
}

// Exact two-word fixed-point split of one coordinate (vqb200_internal.h
// fixed_plan): x * 2^s = hi + lo * 2^-t, hi the integer part of |x| 2^s, lo
// the remainder in units of 2^-t, both carrying x's sign.  Pure integer work
// on the IEEE fields; exact whenever x has no set bit below 2^-(s + t) (the
// column's colstats decide that before any pass runs).
__device__ __forceinline__ void split_fixed_slow(unsigned u, int s, int t, long long& hi, long long& lo) {
  const unsigned E = (u >> 23) & 0xffu;
  unsigned long long m = u & 0x7fffffu;
  int e0 = -149;
  if (E) {
    m |= 0x800000u;
    e0 = (int)E - 150;
  }
  long long h = 0, l = 0;
  if (m) {
    const int k = e0 + s;  // x = m 2^e0, so |x| 2^s = m 2^k
    if (k >= 0) {
      h = (long long)(m << k);  // < 2^61 by the choice of s
    } else {
      const int nk = -k;
      const unsigned long long rem = nk >= 64 ? m : (m & ((1ull << nk) - 1));
      h = nk >= 64 ? 0 : (long long)(m >> nk);
      const int sh = t - nk;  // rem < 2^nk, so rem 2^sh < 2^t
      l = sh >= 0 ? (long long)(rem << sh) : (sh > -64 ? (long long)(rem >> -sh) : 0);
    }
    if (u >> 31) {
      h = -h;
      l = -l;
    }
  }
  hi = h;
  lo = l;
}
// the common case of split_fixed for float32: zero, or a normal value that is
// an integer multiple of the column's grid 2^-s (no low word); false = take
// the general split
__device__ __forceinline__ bool split_fast(float x, int s, long long& h) {
  const unsigned u = __float_as_uint(x);
  const int E = (int)((u >> 23) & 0xffu);
  const int k = E - 150 + s;
  const long long v = (long long)((u & 0x7fffffu) | 0x800000u) << (k & 63);
  const bool zero = (u << 1) == 0;
  h = zero ? 0 : ((int)u < 0 ? -v : v);
  return zero || (E != 0 && k >= 0);
}
__device__ __forceinline__ bool split_fast(double x, int s, long long& h) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  const int E = (int)((u >> 52) & 0x7ffu);
  const int k = E - 1075 + s;
  const long long v = (long long)((u & 0xfffffffffffffull) | (1ull << 52)) << (k & 63);
  const bool zero = (u << 1) == 0;
  h = zero ? 0 : ((long long)u < 0 ? -v : v);
  return zero || (E != 0 && k >= 0);
}
__device__ __forceinline__ void split_fixed(float x, int s, int t, long long& hi, long long& lo) {
  const unsigned u = __float_as_uint(x);
  const int k = (int)((u >> 23) & 0xffu) - 150 + s;
  if (((u >> 23) & 0xffu) != 0 && k >= 0) {
    // the usual case: a normal float32 that is an integer multiple of the
    // column's grid 2^-s (k < 61 - 23 by the choice of s): no low word
    const long long h = (long long)((u & 0x7fffffu) | 0x800000u) << k;
    hi = (u >> 31) ? -h : h;
    lo = 0;
    return;
  }
  split_fixed_slow(u, s, t, hi, lo);
}
__device__ __forceinline__ void split_fixed(double x, int s, int t, long long& hi, long long& lo) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  const unsigned E = (unsigned)((u >> 52) & 0x7ffu);
  unsigned long long m = u & 0xfffffffffffffull;
  int e0 = -1074;
  if (E) {
    m |= 1ull << 52;
    e0 = (int)E - 1075;
  }
  long long h = 0, l = 0;
  if (m) {
    const int k = e0 + s;
    if (k >= 0) {
      h = (long long)(m << k);
    } else {
      const int nk = -k;
      const unsigned long long rem = nk >= 64 ? m : (m & ((1ull << nk) - 1));
      h = nk >= 64 ? 0 : (long long)(m >> nk);
      const int sh = t - nk;
      l = sh >= 0 ? (long long)(rem << sh) : (sh > -64 ? (long long)(rem >> -sh) : 0);
    }
    if (u >> 63) {
      h = -h;
      l = -l;
    }
  }
  hi = h;
  lo = l;
}

// low words are rare for float32 data (only coordinates with bits below the
// column's 2^-s_l): added straight into the exchange buffer's lo section
// (64-bit global atomics; integer adds commute, so still deterministic)
__device__ __forceinline__ void add_lo(const KernelArgs& a, long long cell, int l, long long lo) {
  if (lo) atomicAdd(reinterpret_cast<unsigned long long*>(a.ex.lo() + cell * a.dim + l), (unsigned long long)lo);
}

// (hi 2^t + lo) 2^e rounded once to the nearest double (ties to even): the
// exact two-word cell sum as the FP64 numerator of the centroid
__device__ __forceinline__ double fixed_to_double(long long hi, long long lo, int t, int e) {
  __int128 T = ((__int128)hi << t) + (__int128)lo;
  const bool neg = T < 0;
  unsigned __int128 M = neg ? (unsigned __int128)(-T) : (unsigned __int128)T;
  if (M == 0) return 0.0;
  const unsigned long long mh = (unsigned long long)(M >> 64), ml = (unsigned long long)M;
  const int p = mh ? 127 - __clzll((long long)mh) : 63 - __clzll((long long)ml);  // top bit
  double d;
  if (p <= 52) {
    d = (double)ml;
    d = ldexp(d, e);
  } else {
    const int sh = p - 52;
    unsigned long long mant = (unsigned long long)(M >> sh);
    const unsigned __int128 rem = M & ((((unsigned __int128)1) << sh) - 1);
    const unsigned __int128 half = ((unsigned __int128)1) << (sh - 1);
    if (rem > half || (rem == half && (mant & 1))) ++mant;  // 2^53 after a carry is still exact
    d = ldexp((double)mant, sh + e);
  }
  return neg ? -d : d;
}

// ---------------------------------------------------------------------------
// prep: centred FP32 staging of the current FP64 codebook
// ---------------------------------------------------------------------------

__global__ void prep_codebook_kernel(KernelArgs a) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = st->size;
  const int dim = a.dim, cdim = a.cdim;  // codevectors zero-padded to the candidate width
  const double* cb = a.cb[st->cur];
  const long long kpad = (a.kmax + 3) / 4 * 4;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < kpad;
       k += (long long)gridDim.x * blockDim.x) {
    float* w = a.w + k * cdim;
    if (k < K) {
      double n = 0.0;
      for (int l = 0; l < cdim; ++l) {
        float c = l < dim ? (float)(cb[k * dim + l] - (double)a.mu[l]) : 0.0f;
        n += (double)c * (double)c;
        w[l] = -2.0f * c;
      }
      a.nrm[k] = (float)n;
      stage_tc_row(a, k, w, n);
    } else {
      for (int l = 0; l < cdim; ++l) w[l] = 0.0f;
      a.nrm[k] = INFINITY;  // padding never wins
    }
  }
}

cudaError_t launch_prep_codebook(const KernelArgs& a, cudaStream_t s) {
  long long kpad = (a.kmax + 3) / 4 * 4;
  int blocks = (int)((kpad + 255) / 256);
  if (blocks > 1024) blocks = 1024;
  return launch_k(prep_codebook_kernel, blocks, 256, 0, s, a);
}

// ---------------------------------------------------------------------------
// assign_fast: FP32 candidate pass with a certified error band
// ---------------------------------------------------------------------------

template <int L>
struct FastCfg;
#ifndef VQB_FAST16_NT
#define VQB_FAST16_NT 512
#define VQB_FAST16_R 4
#endif
template <>
struct FastCfg<16> {
  static constexpr int NT = VQB_FAST16_NT, R = VQB_FAST16_R, TK = 1024;
};
template <>
struct FastCfg<32> {
  static constexpr int NT = 256, R = 2, TK = 512;
};
template <>
struct FastCfg<64> {
  static constexpr int NT = 256, R = 2, TK = 256;
};

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("VQB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool fast_dim_supported(int dim) { return dim == 16 || dim == 32 || dim == 64; }

// integer environment switch (A/B timing), read once per name
static int getenv_flag(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// candidate widths with a small-codebook kernel (assign_small_kernel), which
// takes the passes with K < kSmallK
constexpr int kSmallK = 64;
// (the kernel is written for T = L / 16 lanes per row; at L = 64 it measured no
// faster than assign_fast_kernel at K = 2 and 1.6x slower at K = 32 -- cfg3,
// profiles/r02_assign_small_ab.txt -- so only L = 16 takes it)
__host__ __device__ constexpr bool small_dim(int L) { return L == 16; }

template <int L, int TK>
struct TileStream {
  // W tile [TK][L] then norms [TK]; two buffers.
  static constexpr size_t kWBytes = (size_t)TK * L * sizeof(float);
  static constexpr size_t kBufBytes = kWBytes + (size_t)TK * sizeof(float);
};

// Process rows assigned to this thread in one chunk: R rows, strided by NT.
// DIFF: candidate values in DIFFERENCE form, v_j = sum_l (y~_l - c~_l)^2 (the
// distance itself, two FMA-pipe operations per dimension), instead of the
// expanded ||c~_j||^2 - 2 y~.c~_j.  Its error is relative to the distance, not
// to ||y~||^2, so rows whose distance is small against their norm (image
// blocks with a large mean) certify instead of queueing: the kernel takes it
// for K < kSmallK at L >= 32, where the extra FMAs are cheap and the expanded
// form queued ~30 % of cfg3's rows.
template <int L, int NT, int TK, int R, bool PACKED, bool DIFF = false>
__device__ __forceinline__ void assign_chunk(const KernelArgs& a, long long row0, long long row_end,
                                             int K, int ntiles, float* smem, uint64_t* bars,
                                             long long& seq, long long seq_total) {
  const int tid = threadIdx.x;
  float y[R][L];
  float q[R];
  bool valid[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    long long row = row0 + tid + (long long)r * NT;
    valid[r] = row < row_end;
    q[r] = 0.f;
    const float4* src = reinterpret_cast<const float4*>(a.xc + (valid[r] ? row : row0) * L);
#pragma unroll
    for (int v = 0; v < L / 4; ++v) {
      float4 t = __ldg(src + v);
      y[r][4 * v + 0] = __fsub_rn(t.x, a.mu[4 * v + 0]);
      y[r][4 * v + 1] = __fsub_rn(t.y, a.mu[4 * v + 1]);
      y[r][4 * v + 2] = __fsub_rn(t.z, a.mu[4 * v + 2]);
      y[r][4 * v + 3] = __fsub_rn(t.w, a.mu[4 * v + 3]);
    }
#pragma unroll
    for (int l = 0; l < L; ++l) q[r] = fmaf(y[r][l], y[r][l], q[r]);
  }
  float m1[R], m2[R];
  int i1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    m1[r] = INFINITY;
    m2[r] = INFINITY;
    i1[r] = 0;
  }
  using TS = TileStream<L, TK>;
  for (int t = 0; t < ntiles; ++t) {
    const int buf = (ntiles == 1) ? 0 : (int)(seq & 1);
    if (ntiles > 1) mbar_wait(&bars[buf], (uint32_t)((seq >> 1) & 1));
    const float* sW = reinterpret_cast<const float*>(reinterpret_cast<const char*>(smem) +
                                                     buf * TS::kBufBytes);
    const float* sN = reinterpret_cast<const float*>(reinterpret_cast<const char*>(sW) + TS::kWBytes);
    const int jbase = t * TK;
    const int cnt = min(TK, K - jbase);
    if constexpr (PACKED && (R % 2 == 0)) {
      // FFMA2: row pairs share one instruction; 8 issue slots per 16-dim eval pair
      constexpr int P = R / 2;
      unsigned long long y2[P][L];
#pragma unroll
      for (int p = 0; p < P; ++p)
#pragma unroll
        for (int l = 0; l < L; ++l) y2[p][l] = pack2(y[2 * p][l], y[2 * p + 1][l]);
#pragma unroll 2
      for (int j = 0; j < cnt; ++j) {
        const float4* wj = reinterpret_cast<const float4*>(sW + j * L);
        const float nj = sN[j];
        const unsigned long long n2 = pack2(nj, nj);
        unsigned long long v2[P];
#pragma unroll
        for (int p = 0; p < P; ++p) v2[p] = DIFF ? pack2(0.f, 0.f) : n2;
        const unsigned long long half2 = pack2(0.5f, 0.5f);
#pragma unroll
        for (int c = 0; c < L / 4; ++c) {
          const float4 t4 = wj[c];
          const float w[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const unsigned long long w2 = pack2(w[q], w[q]);
#pragma unroll
            for (int p = 0; p < P; ++p) {
              if constexpr (DIFF) {
                // y~ - c~ = y~ + 0.5 w (w = -2 c~: the halving is exact, one rounding)
                const unsigned long long d2 = ffma2(half2, w2, y2[p][c * 4 + q]);
                v2[p] = ffma2(d2, d2, v2[p]);
              } else {
                v2[p] = ffma2(y2[p][c * 4 + q], w2, v2[p]);
              }
            }
          }
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
          float va, vb;
          unpack2(v2[p], va, vb);
          const float vv[2] = {va, vb};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = 2 * p + h;
            const float n2r = fminf(m2[r], fmaxf(m1[r], vv[h]));
            const bool pr = vv[h] < m1[r];
            m1[r] = fminf(m1[r], vv[h]);
            i1[r] = pr ? jbase + j : i1[r];
            m2[r] = n2r;
          }
        }
      }
    } else {
#pragma unroll 2
    for (int j = 0; j < cnt; ++j) {
      const float4* wj = reinterpret_cast<const float4*>(sW + j * L);
      float v[R];
      const float nj = sN[j];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = DIFF ? 0.f : nj;
#pragma unroll
      for (int c = 0; c < L / 16; ++c) {
        float w[16];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          float4 t4 = wj[c * 4 + p];
          w[4 * p + 0] = t4.x;
          w[4 * p + 1] = t4.y;
          w[4 * p + 2] = t4.z;
          w[4 * p + 3] = t4.w;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
          for (int l = 0; l < 16; ++l) {
            if constexpr (DIFF) {
              const float d = fmaf(0.5f, w[l], y[r][c * 16 + l]);
              v[r] = fmaf(d, d, v[r]);
            } else {
              v[r] = fmaf(w[l], y[r][c * 16 + l], v[r]);
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float vv = v[r];
        const float n2 = fminf(m2[r], fmaxf(m1[r], vv));
        const bool p = vv < m1[r];
        m1[r] = fminf(m1[r], vv);
        i1[r] = p ? jbase + j : i1[r];
        m2[r] = n2;
      }
    }
    }
    if (ntiles > 1) {
      __syncthreads();  // every warp is done with buffer `buf`
      if (tid == 0 && seq + 2 < seq_total) {
        const long long ns = seq + 2;
        const int nt = (int)(ns % ntiles);
        const int ncnt = min(TK, K - nt * TK);
        const uint32_t wbytes = (uint32_t)ncnt * L * sizeof(float);
        const uint32_t nbytes = (uint32_t)((ncnt + 3) / 4 * 4) * sizeof(float);
        float* dW = reinterpret_cast<float*>(reinterpret_cast<char*>(smem) + buf * TS::kBufBytes);
        float* dN = reinterpret_cast<float*>(reinterpret_cast<char*>(dW) + TS::kWBytes);
        mbar_arrive_expect_tx(&bars[buf], wbytes + nbytes);
        bulk_g2s(dW, a.w + (long long)nt * TK * L, wbytes, &bars[buf]);
        bulk_g2s(dN, a.nrm + (long long)nt * TK, nbytes, &bars[buf]);
      }
      ++seq;
    }
  }
  // Certification.  With y~ = fl(x - mu) and the centred FP32 codebook, the
  // computed v_j = fl-chain(||c~_j||^2 - 2 y~.c~_j) differs from the exact
  // ||x - c_j||^2 - ||y~||^2 by at most
  //   (L+3) u S^2 + 2.5 u sqrt(D) S,   S = 2||y~|| + sqrt(D) (+ slack),
  // (u = 2^-24; FMA-chain, norm rounding, centring and FP32 codebook
  // rounding; ||c~_j|| <= ||y~|| + sqrt(D_j)), plus the FP64 reference's own
  // rounding (~1e-14 D).  If the top-2 gap exceeds 3x that bound (2 rows'
  // worth x 1.5 safety) the FP32 winner is the reference's winner; otherwise
  // the row is re-ranked in exact FP64.  NaN / inf propagate to "flag".
  const float u = 5.9604645e-8f;
  const int lane = tid & 31;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    long long row = row0 + tid + (long long)r * NT;
    bool ok = false;
    float thr = NAN;
    if (valid[r]) {
      const float yn = sqrtf(q[r]);
      // distance of the runner-up: m2 itself in difference form
      const float d2 = fmaxf(DIFF ? m2[r] : m2[r] + q[r], 0.f);
      const float sd = sqrtf(d2) * 1.01f + 1.0f;
      const float S = 2.02f * yn + sd;
      const float E = (float)(L + 3) * u * S * S + 2.5f * u * sd * S + 1e-14f * S * S;
      if constexpr (DIFF) {
        // t_l = fl(y~_l - c~_l) differs from x_l - c_l by e_l, |e_l| <= u (|y~_l|
        // + |c~_l| + |t_l|) (centring, FP32 codebook rounding, the difference),
        // so ||e|| <= 2 u (||y~|| + sqrt T) with T = sum t^2, and the FMA chain
        // of L non-negative terms adds at most (L + 1) u T:
        //   |v - d| <= (L + 3) u sd^2 + 4.1 u sd (yn + sd) =: Ed   (sd >= sqrt of
        // every distance up to the runner-up's; v - Ed(v) grows with v, so the
        // runner-up's bound covers every farther codevector).  Certified iff
        // the gap exceeds 3 Ed (two values' worth x 1.5, as above).
        const float Ed = (float)(L + 3) * u * sd * sd + 4.1f * u * sd * (yn + sd) + 1e-14f * S * S;
        const float bandd = 3.0f * Ed + input_band(rin_of(a, row), m1[r], 3.0f * Ed);
        ok = (m2[r] - m1[r]) > bandd;
        // the re-rank rescans in the EXPANDED arithmetic (v = d - ||y~||^2 up
        // to E): the reference's winner has d <= m1 + Ed, hence v <= m1 - q +
        // Ed + E (+ the rounding of q and of the subtraction)
        const float bande = 3.0f * E + input_band(rin_of(a, row), m1[r], 3.0f * E);
        thr = (m1[r] - q[r]) + bande + bandd + (float)(L + 8) * u * (q[r] + fabsf(m1[r]));
      } else {
      // float64 rows: + the band of their float32 rounding (input_band)
      const float band = 3.0f * E + input_band(rin_of(a, row), m1[r] + q[r], 3.0f * E);
      ok = (m2[r] - m1[r]) > band;
      thr = m1[r] + band;  // shortlist band (shortlist_kernel)
      }
      a.idx[row] = i1[r];
      if (ok && a.dists) store_dist(a, row, row_dist<L>(a, row, a.cb[a.st->cur], i1[r]));
    }
    const bool flag = valid[r] && !ok;
    const unsigned mask = __ballot_sync(0xffffffffu, flag);
    if (mask) {
      int base = 0;
      const int leader = __ffs(mask) - 1;
      if (lane == leader) base = atomicAdd(&a.st->flag_count, __popc(mask));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (flag) {
        const int pos = base + __popc(mask & ((1u << lane) - 1u));
        a.flags[pos] = (int)row;
        a.flag_thr[pos] = thr;
      }
    }
  }
}

template <int L, bool PACKED>
__global__ void __launch_bounds__(FastCfg<L>::NT, 1) assign_fast_kernel(KernelArgs a) {
  pdl_wait();
  constexpr int NT = FastCfg<L>::NT, R = FastCfg<L>::R, TK = FastCfg<L>::TK;
  using TS = TileStream<L, TK>;
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = st->size;
  if (a.tcb && tc_handles(st, K)) return;  // assign_tc runs this pass
  if (small_dim(L) && a.small_on && K < kSmallK) return;  // assign_small_kernel runs this pass
  const int ntiles = (K + TK - 1) / TK;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* smem = reinterpret_cast<float*>(smem_raw);
  __shared__ __align__(8) uint64_t bars[2];

  // contiguous, balanced row range for this block (within [r0, r1))
  const long long n = a.r1 - a.r0;
  const long long lo = a.r0 + n * blockIdx.x / gridDim.x;
  const long long hi = a.r0 + n * (blockIdx.x + 1) / gridDim.x;
  const long long rows = hi - lo;
  const long long per_chunk = (long long)NT * R;
  const long long full = rows / per_chunk;
  const long long rem = rows - full * per_chunk;
  const long long nchunks = full + (rem > 0 ? 1 : 0);
  const long long seq_total = (ntiles > 1) ? nchunks * ntiles : 1;

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (nchunks == 0) return;
  if (threadIdx.x == 0) {
    const int first = (ntiles > 1) ? 2 : 1;
    for (int s = 0; s < first && s < seq_total; ++s) {
      const int t = s % ntiles;
      const int cnt = min(TK, K - t * TK);
      const uint32_t wbytes = (uint32_t)cnt * L * sizeof(float);
      const uint32_t nbytes = (uint32_t)((cnt + 3) / 4 * 4) * sizeof(float);
      float* dW = reinterpret_cast<float*>(smem_raw + s * TS::kBufBytes);
      float* dN = reinterpret_cast<float*>(smem_raw + s * TS::kBufBytes + TS::kWBytes);
      mbar_arrive_expect_tx(&bars[s], wbytes + nbytes);
      bulk_g2s(dW, a.w + (long long)t * TK * L, wbytes, &bars[s]);
      bulk_g2s(dN, a.nrm + (long long)t * TK, nbytes, &bars[s]);
    }
  }
  if (ntiles == 1) mbar_wait(&bars[0], 0);

  long long seq = 0;
  const bool diff = L >= 32 && K < kSmallK && a.diff_on;  // difference-form values (assign_chunk)
  for (long long c = 0; c < full; ++c) {
    if (diff)
      assign_chunk<L, NT, TK, R, PACKED, (L >= 32)>(a, lo + c * per_chunk, hi, K, ntiles, smem, bars, seq,
                                                    seq_total);
    else
      assign_chunk<L, NT, TK, R, PACKED>(a, lo + c * per_chunk, hi, K, ntiles, smem, bars, seq,
                                         seq_total);
  }
  if (rem > 0 && diff) {
    // tail chunk in difference form: the full row count per thread (rows past
    // the range are masked)
    assign_chunk<L, NT, TK, R, PACKED, (L >= 32)>(a, lo + full * per_chunk, hi, K, ntiles, smem, bars, seq,
                                                  seq_total);
  } else if (rem > 0) {
    // tail chunk: only as many rows per thread as needed (no wave tail)
    const long long row0 = lo + full * per_chunk;
    int rr = (int)((rem + NT - 1) / NT);
    if (PACKED && (rr & 1)) ++rr;  // row pairs
    if (rr >= 4)
      assign_chunk<L, NT, TK, (R >= 4 ? 4 : R), PACKED>(a, row0, hi, K, ntiles, smem, bars, seq,
                                                        seq_total);
    else if (rr == 3)
      assign_chunk<L, NT, TK, (R >= 3 ? 3 : R), PACKED>(a, row0, hi, K, ntiles, smem, bars, seq,
                                                        seq_total);
    else if (rr == 2)
      assign_chunk<L, NT, TK, (R >= 2 ? 2 : R), PACKED>(a, row0, hi, K, ntiles, smem, bars, seq,
                                                        seq_total);
    else
      assign_chunk<L, NT, TK, 1, PACKED>(a, row0, hi, K, ntiles, smem, bars, seq, seq_total);
  }
}

// ---------------------------------------------------------------------------
// Small codebooks (K < kSmallK, the sizes the tensor-core pass leaves to the
// FP32 kernels): candidate pass with ONE ROW PER THREAD, rows staged through
// shared memory.  assign_fast_kernel reads a row per lane straight from
// global memory (4 x LDG.128 at a 64-byte stride: 16 cache lines per warp
// instruction), reads it again for the FP64 winner distance and gathers the
// winner's codevector from global memory; at K = 2..32 that load pattern --
// not the arithmetic -- set its time (cfg4: 0.46-0.89 ms against 0.18 ms of
// HBM time; more CTAs per SM, L1 / L2 prefetches did not move it).  Here a
// tile of 256 rows is fetched with fully coalesced 16-byte loads one tile
// ahead (registers), parked in shared memory with a padded row stride (each
// thread then reads its own row in 4-wavefront LDS.128s, again for the exact
// FP64 distance), and the FP64 codebook (<= 63 rows) sits in shared memory
// too.  Distances as FFMA2 over dimension pairs; assign_chunk's band and
// re-rank queue.
// Reference: _kernels.assign_range (_kernels.py:18-36).
// ---------------------------------------------------------------------------
constexpr int kSmallNT = 256;
#ifndef VQB_SMALL_MINB
#define VQB_SMALL_MINB 3
#endif
constexpr int kSmallMinB = VQB_SMALL_MINB;  // CTAs per SM the kernel is compiled for (A/B builds: 4)
// T = L / 16 adjacent lanes share a row, 16 dimensions each (a row of 64
// dimensions in one thread's registers would leave 8 warps per SM); their
// partial sums meet in a butterfly, so every lane of a row holds the same
// value bits and takes the same top-2 decisions.  Shared-memory layouts are
// chosen so that a quarter-warp's LDS.128s fall on distinct bank groups: the
// row tile as T sub-tiles (16 dimensions of every row, 20-word row stride,
// sub-tiles skewed by 32 / T words), the FP32 codebook with a 20-word stride
// per 16-dimension slice.
template <int L>
struct SmallSmem {
  static constexpr int T = L / 16;           // lanes per row
  static constexpr int RT = kSmallNT / T;    // rows per tile
  static constexpr int SUB = RT * 20 + (T > 1 ? 32 / T : 0);  // sub-tile stride (words)
  static constexpr int WSS = T > 1 ? 20 : 16;                 // codebook slice stride (words)
  static constexpr int WSJ = T * WSS;                         // codevector stride (words)
  static constexpr int CS = L + 2;  // FP64 codevector stride (doubles): <= 2-way conflicts across winners
  float x[2][T * SUB];
  double cb[kSmallK * CS];
  float w[kSmallK * WSJ];
  float nrm[kSmallK];
  float mu[L];
};

template <int L>
__global__ void __launch_bounds__(kSmallNT, L == 16 ? kSmallMinB : 2) assign_small_kernel(KernelArgs a) {
  pdl_wait();
  DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = st->size;
  if (K >= kSmallK || (a.tcb && tc_handles(st, K))) return;  // assign_fast / assign_tc take this pass
  using SM = SmallSmem<L>;
  constexpr int NT = kSmallNT, T = SM::T, RT = SM::RT, CS = SM::CS, CH = L / 4;  // CH: 16-byte chunks per row
  // difference-form values at L >= 32 (assign_chunk's DIFF: image blocks with a
  // large mean certify instead of queueing)
  constexpr bool DIFF = L >= 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31;
  const int rloc = tid / T, sub = tid % T;  // this lane's row of the tile and its 16-dimension slice
  // the staged row serves the winner distance when the candidate rows ARE
  // the rows the reference sees (float32 rows of width L)
  const bool regs_exact = a.x32 != nullptr && a.x64 == nullptr && a.dim == L && a.xc == a.x32;
  const double* cbg = a.cb[st->cur];
  const bool euclid = st->metric == kEuclidean;
  for (int e = tid; e < K * L; e += NT) {
    const int j = e / L, l = e % L;
    sm.w[j * SM::WSJ + (l / 16) * SM::WSS + l % 16] = a.w[e];
  }
  for (int e = tid; e < K; e += NT) sm.nrm[e] = a.nrm[e];
  if (tid < L) sm.mu[tid] = a.mu[tid];
  if (regs_exact)
    for (int e = tid; e < K * L; e += NT) sm.cb[(e / L) * CS + e % L] = cbg[e];

  const long long n = a.r1 - a.r0;
  const long long lo = a.r0 + n * blockIdx.x / gridDim.x;
  const long long hi = a.r0 + n * (blockIdx.x + 1) / gridDim.x;
  const long long ntile = (hi - lo + RT - 1) / RT;
  float4 nxt[4];  // RT * CH = 4 * NT chunks per tile for every L
  auto fetch = [&](long long t) {  // tile t's chunks tid, tid + NT, ...: consecutive lanes, consecutive 16 bytes
    const long long r0 = lo + t * RT;
    const float4* src = reinterpret_cast<const float4*>(a.xc + r0 * L);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = tid + k * NT;
      nxt[k] = (t < ntile && r0 + q / CH < hi) ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto xaddr = [&](int buf, int r, int cc) -> float* {  // chunk cc of row r of the staged tile
    return &sm.x[buf][(cc / 4) * SM::SUB + r * 20 + (cc % 4) * 4];
  };
  auto park = [&](int buf) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = tid + k * NT;
      *reinterpret_cast<float4*>(xaddr(buf, q / CH, q % CH)) = nxt[k];
    }
  };
  if (ntile > 0) {
    fetch(0);
    park(0);
    fetch(1);
  }
  __syncthreads();
  const float u = 5.9604645e-8f;
  for (long long t = 0; t < ntile; ++t) {
    const int buf = (int)(t & 1);
    const long long row = lo + t * RT + rloc;
    const bool valid = row < hi && sub == 0;  // one lane per row certifies and stores
    // y~ = fl(x - mu) packed in dimension pairs for FFMA2, ||y~||^2 as FMA
    // chains (per slice, then the butterfly)
    unsigned long long y2[8];
    float q = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float4 v = *reinterpret_cast<const float4*>(xaddr(buf, rloc, sub * 4 + c));
      const float4 mu4 = *reinterpret_cast<const float4*>(sm.mu + sub * 16 + c * 4);
      const float y0 = __fsub_rn(v.x, mu4.x), y1 = __fsub_rn(v.y, mu4.y);
      const float y2f = __fsub_rn(v.z, mu4.z), y3 = __fsub_rn(v.w, mu4.w);
      q = fmaf(y0, y0, q);
      q = fmaf(y1, y1, q);
      q = fmaf(y2f, y2f, q);
      q = fmaf(y3, y3, q);
      y2[2 * c] = pack2(y0, y1);
      y2[2 * c + 1] = pack2(y2f, y3);
    }
#pragma unroll
    for (int o = 1; o < T; o <<= 1) q = __fadd_rn(q, __shfl_xor_sync(0xffffffffu, q, o));
    // tile t + 1 into the other buffer (its readers passed the barrier that
    // ended iteration t - 1), tile t + 2 into registers; this tile's rows
    // stay in their buffer for the winner distance below
    park(buf ^ 1);
    fetch(t + 2);
    float m1 = INFINITY, m2 = INFINITY;
    int i1 = 0;
    const unsigned long long half2 = pack2(0.5f, 0.5f);
#pragma unroll 2
    for (int j = 0; j < K; ++j) {
      // expanded form: v_j = ||c~_j||^2 - 2 y~.c~_j; difference form:
      // sum (y~ - c~_j)^2 -- two interleaved FMA chains per slice (even / odd
      // dimensions, one FFMA2 per pair), added, then the butterfly over the
      // row's lanes: at most 8 + 1 + log2 T + 1 roundings on a path, inside
      // the band's (L + 3) u term
      unsigned long long v2 = pack2(DIFF || sub != 0 ? 0.f : sm.nrm[j], 0.f);
      const float4* wj = reinterpret_cast<const float4*>(sm.w + j * SM::WSJ + sub * SM::WSS);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 w4 = wj[c];  // one address per slice: a broadcast
        if constexpr (DIFF) {
          // y~ - c~ = y~ + 0.5 w (w = -2 c~: the halving is exact, one rounding)
          const unsigned long long da = ffma2(half2, pack2(w4.x, w4.y), y2[2 * c]);
          const unsigned long long db = ffma2(half2, pack2(w4.z, w4.w), y2[2 * c + 1]);
          v2 = ffma2(da, da, v2);
          v2 = ffma2(db, db, v2);
        } else {
          v2 = ffma2(pack2(w4.x, w4.y), y2[2 * c], v2);
          v2 = ffma2(pack2(w4.z, w4.w), y2[2 * c + 1], v2);
        }
      }
      float va, vb;
      unpack2(v2, va, vb);
      float v = __fadd_rn(va, vb);
#pragma unroll
      for (int o = 1; o < T; o <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
      const float n2 = fminf(m2, fmaxf(m1, v));
      const bool pr = v < m1;
      m1 = fminf(m1, v);
      i1 = pr ? j : i1;
      m2 = n2;
    }
    // certification: assign_chunk's bands (expanded / difference form)
    bool ok = false;
    float thr = NAN;
    if (valid) {
      const float yn = sqrtf(q);
      const float d2 = fmaxf(DIFF ? m2 : m2 + q, 0.f);
      const float sd = sqrtf(d2) * 1.01f + 1.0f;
      const float S = 2.02f * yn + sd;
      const float E = (float)(L + 3) * u * S * S + 2.5f * u * sd * S + 1e-14f * S * S;
      if constexpr (DIFF) {
        const float Ed = (float)(L + 3) * u * sd * sd + 4.1f * u * sd * (yn + sd) + 1e-14f * S * S;
        const float bandd = 3.0f * Ed + input_band(rin_of(a, row), m1, 3.0f * Ed);
        ok = (m2 - m1) > bandd;
        const float bande = 3.0f * E + input_band(rin_of(a, row), m1, 3.0f * E);
        thr = (m1 - q) + bande + bandd + (float)(L + 8) * u * (q + fabsf(m1));
      } else {
        const float band = 3.0f * E + input_band(rin_of(a, row), m1 + q, 3.0f * E);
        ok = (m2 - m1) > band;
        thr = m1 + band;
      }
      a.idx[row] = i1;
      if (ok && a.dists) {
        double d = 0.0;
        if (regs_exact) {
          // the reference's arithmetic (_kernels.py:25-29) on the staged row
          const double2* c2 = reinterpret_cast<const double2*>(sm.cb + i1 * CS);
#pragma unroll 4
          for (int c = 0; c < CH; ++c) {
            const float4 xv = *reinterpret_cast<const float4*>(xaddr(buf, rloc, c));
            const double2 ca = c2[2 * c], cb2 = c2[2 * c + 1];
            const double d0 = __dsub_rn((double)xv.x, ca.x);
            d = __dadd_rn(d, __dmul_rn(d0, d0));
            const double d1 = __dsub_rn((double)xv.y, ca.y);
            d = __dadd_rn(d, __dmul_rn(d1, d1));
            const double d2v = __dsub_rn((double)xv.z, cb2.x);
            d = __dadd_rn(d, __dmul_rn(d2v, d2v));
            const double d3 = __dsub_rn((double)xv.w, cb2.y);
            d = __dadd_rn(d, __dmul_rn(d3, d3));
          }
        } else {
          d = row_dist<L>(a, row, cbg, i1);
        }
        a.dists[row] = euclid ? sqrt(d) : d;
      }
    }
    const bool flag = valid && !ok;
    const unsigned mask = __ballot_sync(0xffffffffu, flag);
    if (mask) {
      int base = 0;
      const int leader = __ffs(mask) - 1;
      if (lane == leader) base = atomicAdd(&st->flag_count, __popc(mask));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (flag) {
        const int pos = base + __popc(mask & ((1u << lane) - 1u));
        a.flags[pos] = (int)row;
        a.flag_thr[pos] = thr;
      }
    }
    __syncthreads();
  }
}

template <int L>
static cudaError_t launch_small_L(const KernelArgs& a, int sms, cudaStream_t s) {
  const size_t smem = sizeof(SmallSmem<L>);
  cudaError_t e = cudaFuncSetAttribute(assign_small_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const long long n = a.r1 - a.r0;
  long long grid = (long long)sms * (L == 16 ? kSmallMinB : 2);
  const long long tiles = (n + SmallSmem<L>::RT - 1) / SmallSmem<L>::RT;
  if (grid > tiles) grid = tiles > 0 ? tiles : 1;
  return launch_k(assign_small_kernel<L>, (unsigned)grid, kSmallNT, smem, s, a);
}

static bool packed_default() {
  // VQB_ASSIGN=ffma selects the scalar-FFMA candidate loop (A/B measurements)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VQB_ASSIGN");
    v = (e && strcmp(e, "ffma") == 0) ? 0 : 1;
  }
  return v == 1;
}

template <int L, bool PACKED>
static cudaError_t launch_fast_LP(const KernelArgs& a, int sms, cudaStream_t s) {
  constexpr int TK = FastCfg<L>::TK;
  using TS = TileStream<L, TK>;
  const int ntiles_max = (int)((a.kmax + TK - 1) / TK);
  const size_t smem = TS::kBufBytes * (ntiles_max > 1 ? 2 : 1);
  cudaError_t e = cudaFuncSetAttribute(assign_fast_kernel<L, PACKED>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = launch_k(assign_fast_kernel<L, PACKED>, sms, FastCfg<L>::NT, smem, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int L>
static cudaError_t launch_fast_L(const KernelArgs& a, int sms, cudaStream_t s) {
  return packed_default() ? launch_fast_LP<L, true>(a, sms, s) : launch_fast_LP<L, false>(a, sms, s);
}

// ---------------------------------------------------------------------------
// exact FP64 rows: G lanes per row (G = min(32, pow2 >= K)), lanes stride the
// codebook, a lexicographic (d, j) shuffle reduction reproduces the strict-<
// ascending scan.  DIM is a compile-time row length (0 = runtime).
// ---------------------------------------------------------------------------

template <int DIM, typename XT>
__device__ __forceinline__ double ref_dist_regs(const XT (&xr)[DIM], const double* __restrict__ c) {
  double d = 0.0;
#pragma unroll
  for (int c0 = 0; c0 < DIM; c0 += 16) {
    double cr[16];
    const double2* c2 = reinterpret_cast<const double2*>(c + c0);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double2 t = __ldg(c2 + v);
      cr[2 * v] = t.x;
      cr[2 * v + 1] = t.y;
    }
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      const double diff = __dsub_rn((double)xr[c0 + l], cr[l]);
      d = __dadd_rn(d, __dmul_rn(diff, diff));
    }
  }
  return d;
}

template <typename XT, int DIM>
__global__ void __launch_bounds__(256) exact_rows_kernel(KernelArgs a, const XT* __restrict__ X,
                                                         int use_list) {
  pdl_wait();
  // use_list: 0 every row, 1 the assign_fast queue, 2 the shortlist overflow queue
  // T threads per row (T = pow2 >= K, capped at the block): K=2 packs 128
  // rows per block, K >= 256 gives one block per row.  Each thread scans
  // j = t, t+T, ... (ascending) with the reference's strict <, then a
  // lexicographic (d, j) reduction over the T threads.
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = st->size;
  const int dim = DIM ? DIM : a.dim;
  const double* __restrict__ cb = a.cb[st->cur];
  if constexpr (DIM > 0) {
    if (K > 32) {
      // large K: a batch of 8 rows per block shares every codevector load;
      // thread t scans j = t, t + 256, ... for all 8 rows
      constexpr int B = 8;
      __shared__ XT xs[B][DIM];
      __shared__ double s_b[8][B];
      __shared__ int s_j[8][B];
      __shared__ long long s_row[B];
      const int* list = use_list == 2 ? a.flags2 : a.flags;
      const long long count = use_list == 2 ? (long long)st->flag2_count
                              : use_list ? (long long)st->flag_count : a.n;
      for (long long base = (long long)blockIdx.x * B; base < count; base += (long long)gridDim.x * B) {
        if (threadIdx.x < B) {
          const long long i = base + threadIdx.x;
          s_row[threadIdx.x] = i < count ? (use_list ? (long long)list[i] : i) : -1;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < B * DIM; e += blockDim.x) {
          const long long r = s_row[e / DIM];
          xs[e / DIM][e % DIM] = r >= 0 ? X[r * DIM + e % DIM] : (XT)0;
        }
        __syncthreads();
        double best[B];
        int bj[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
          best[b] = INFINITY;
          bj[b] = 0x7fffffff;
        }
        for (int j = threadIdx.x; j < K; j += blockDim.x) {
          const double* c = cb + (long long)j * DIM;
          double d[B];
#pragma unroll
          for (int b = 0; b < B; ++b) d[b] = 0.0;
#pragma unroll
          for (int c0 = 0; c0 < DIM; c0 += 16) {
            double cr[16];
            const double2* c2 = reinterpret_cast<const double2*>(c + c0);
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const double2 q = __ldg(c2 + v);
              cr[2 * v] = q.x;
              cr[2 * v + 1] = q.y;
            }
            // the reference's arithmetic, ascending c (_kernels.py:25-29)
#pragma unroll
            for (int b = 0; b < B; ++b) {
#pragma unroll
              for (int l = 0; l < 16; ++l) {
                const double diff = __dsub_rn((double)xs[b][c0 + l], cr[l]);
                d[b] = __dadd_rn(d[b], __dmul_rn(diff, diff));
              }
            }
          }
#pragma unroll
          for (int b = 0; b < B; ++b)
            if (d[b] < best[b]) {  // ascending j per thread: first minimum kept
              best[b] = d[b];
              bj[b] = j;
            }
        }
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
        for (int b = 0; b < B; ++b) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best[b], off);
            const int oj = __shfl_xor_sync(0xffffffffu, bj[b], off);
            if (ob < best[b] || (ob == best[b] && oj < bj[b])) {
              best[b] = ob;
              bj[b] = oj;
            }
          }
          if (lane == 0) {
            s_b[w][b] = best[b];
            s_j[w][b] = bj[b];
          }
        }
        __syncthreads();
        if (threadIdx.x < B && s_row[threadIdx.x] >= 0) {
          const int b = threadIdx.x;
          double bb = s_b[0][b];
          int jj = s_j[0][b];
          for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
            if (s_b[k][b] < bb || (s_b[k][b] == bb && s_j[k][b] < jj)) {
              bb = s_b[k][b];
              jj = s_j[k][b];
            }
          a.idx[s_row[b]] = (bb < INFINITY) ? jj : 0;  // nothing < inf -> index 0
          store_dist(a, s_row[b], bb);
        }
        __syncthreads();
      }
      return;
    }
  }
  int T = 1;
  while (T < K && T < (int)blockDim.x) T <<= 1;
  const int rpb = blockDim.x / T;
  const int sub = threadIdx.x / T, tl = threadIdx.x % T;
  __shared__ double s_best[8];
  __shared__ int s_bj[8];
  const int* list = use_list == 2 ? a.flags2 : a.flags;
  const long long count = use_list == 2 ? (long long)st->flag2_count
                          : use_list ? (long long)st->flag_count : a.n;
  for (long long base = (long long)blockIdx.x * rpb; base < count; base += (long long)gridDim.x * rpb) {
    const long long i = base + sub;
    const bool valid = i < count;
    const long long row = valid ? (use_list ? (long long)list[i] : i) : 0;
    double best = INFINITY;
    int bj = 0x7fffffff;
    if (valid) {
      const XT* x = X + row * dim;
      if constexpr (DIM > 0) {
        XT xr[DIM];
#pragma unroll
        for (int l = 0; l < DIM; ++l) xr[l] = x[l];
        int j = tl;
        for (; j + T < K; j += 2 * T) {  // two codevectors in flight
          const double d0 = ref_dist_regs<DIM, XT>(xr, cb + (long long)j * DIM);
          const double d1 = ref_dist_regs<DIM, XT>(xr, cb + (long long)(j + T) * DIM);
          if (d0 < best) {
            best = d0;
            bj = j;
          }
          if (d1 < best) {
            best = d1;
            bj = j + T;
          }
        }
        if (j < K) {
          const double d0 = ref_dist_regs<DIM, XT>(xr, cb + (long long)j * DIM);
          if (d0 < best) {
            best = d0;
            bj = j;
          }
        }
      } else {
        for (int j = tl; j < K; j += T) {
          const double d = ref_dist(x, cb + (long long)j * dim, dim);
          if (d < best) {
            best = d;
            bj = j;
          }
        }
      }
    }
    const int seg = T < 32 ? T : 32;
    for (int off = seg >> 1; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
      if (ob < best || (ob == best && oj < bj)) {
        best = ob;
        bj = oj;
      }
    }
    if (T > 32) {  // a row spans T/32 warps: combine them in order
      const int w = threadIdx.x >> 5;
      if ((threadIdx.x & 31) == 0) {
        s_best[w] = best;
        s_bj[w] = bj;
      }
      __syncthreads();
      if (tl == 0) {
        for (int k = w + 1; k < w + T / 32; ++k)
          if (s_best[k] < best || (s_best[k] == best && s_bj[k] < bj)) {
            best = s_best[k];
            bj = s_bj[k];
          }
      }
      __syncthreads();
    }
    if (valid && tl == 0) {
      a.idx[row] = (best < INFINITY) ? bj : 0;  // nothing < inf -> index 0
      store_dist(a, row, best);
    }
  }
}

template <typename XT>
static cudaError_t launch_exact_t(const KernelArgs& a, const XT* X, int use_list, int sms,
                                  cudaStream_t s) {
  const int blocks = sms * 4;
  cudaError_t e;
  switch (a.dim) {
    case 16: e = launch_k(exact_rows_kernel<XT, 16>, blocks, 256, 0, s, a, X, use_list); break;
    case 32: e = launch_k(exact_rows_kernel<XT, 32>, blocks, 256, 0, s, a, X, use_list); break;
    case 64: e = launch_k(exact_rows_kernel<XT, 64>, blocks, 256, 0, s, a, X, use_list); break;
    default: e = launch_k(exact_rows_kernel<XT, 0>, blocks, 256, 0, s, a, X, use_list); break;
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------------------
// shortlist: the queued rows' exact winner from a band of candidates.
//
// A row is queued when its FP32 top-2 gap is within the certified error
// 3E.  The reference's winner j* then satisfies v_j* <= m1 + 3E in the same
// FP32 expanded form (any evaluation order: E bounds every order of the
// length-L FMA chain, and 3E >= 2E + 2x the FP64 reference's own rounding),
// so rescanning the codebook in FP32 and keeping every j with v_j <= m1 + 3E
// yields a shortlist that contains j* and every index tied with it.  Only
// the shortlist is evaluated in the reference's FP64 arithmetic (ascending j,
// strict <: lowest index on ties).  A row whose band holds more than kShort
// candidates (or a non-finite threshold) goes to the full FP64 scan.
// Costs ~L FFMA per codevector instead of 3L FP64 ops.
// ---------------------------------------------------------------------------

template <int L>
struct ShortCfg {
  static constexpr int NT = 256;
  static constexpr int TK = L == 16 ? 1024 : (L == 32 ? 512 : 256);  // 64 KB FP32 tile
  static constexpr size_t kSmem = (size_t)TK * L * 4 + (size_t)TK * 4;
};
constexpr int kShort = 8;

template <int L>
__global__ void __launch_bounds__(256) shortlist_kernel(KernelArgs a) {
  pdl_wait();
  using C = ShortCfg<L>;
  constexpr int NT = C::NT, TK = C::TK;
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const long long count = st->flag_count;
  if (count == 0) return;
  const int K = st->size;
  if (a.tcb && tc_handles(st, K) && count * (long long)K >= kTcShortlistWork) return;  // the TC shortlist runs
  const double* __restrict__ cb = a.cb[st->cur];
  if (count < (long long)gridDim.x * NT) {
    // Few queued rows (e.g. a converged codebook): one warp per row, lanes
    // stride the codebook (j = lane, lane + 32, ...) so the rows' work
    // spreads over every SM; candidates are gathered by ballot in
    // ascending j, then evaluated one per lane in FP64.
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (NT / 32);
    for (long long i = blockIdx.x * (long long)(NT / 32) + (threadIdx.x >> 5); i < count; i += warps) {
      const long long row = a.flags[i];
      const float thr = a.flag_thr[i];
      float y[L];
      const float4* src = reinterpret_cast<const float4*>(a.xc + row * L);
#pragma unroll
      for (int v = 0; v < L / 4; ++v) {
        const float4 t = __ldg(src + v);
        y[4 * v + 0] = __fsub_rn(t.x, a.mu[4 * v + 0]);
        y[4 * v + 1] = __fsub_rn(t.y, a.mu[4 * v + 1]);
        y[4 * v + 2] = __fsub_rn(t.z, a.mu[4 * v + 2]);
        y[4 * v + 3] = __fsub_rn(t.w, a.mu[4 * v + 3]);
      }
      int nc = 0;
      int mine = -1;  // lane c holds the c-th candidate (ascending j)
      for (int jb = 0; jb < K; jb += 32) {
        const int j = jb + lane;
        bool in = false;
        if (j < K) {
          const float4* wj = reinterpret_cast<const float4*>(a.w + (long long)j * L);
          float v0 = __ldg(a.nrm + j), v1 = 0.f;
#pragma unroll
          for (int c = 0; c < L / 4; ++c) {
            const float4 w4 = __ldg(wj + c);
            if (c & 1) {
              v1 = fmaf(w4.x, y[4 * c + 0], v1);
              v1 = fmaf(w4.y, y[4 * c + 1], v1);
              v1 = fmaf(w4.z, y[4 * c + 2], v1);
              v1 = fmaf(w4.w, y[4 * c + 3], v1);
            } else {
              v0 = fmaf(w4.x, y[4 * c + 0], v0);
              v0 = fmaf(w4.y, y[4 * c + 1], v0);
              v0 = fmaf(w4.z, y[4 * c + 2], v0);
              v0 = fmaf(w4.w, y[4 * c + 3], v0);
            }
          }
          in = (v0 + v1) <= thr;
        }
        const unsigned m = __ballot_sync(0xffffffffu, in);
        // lane c picks the c-th candidate overall (ascending j)
        const int before = nc;
        nc += __popc(m);
        if (lane >= before && lane < nc && lane < 32) {
          // position of the (lane - before)-th set bit of m
          unsigned mm = m;
          for (int k = 0; k < lane - before; ++k) mm &= mm - 1;
          mine = jb + __ffs(mm) - 1;
        }
      }
      if (nc == 0 || nc > kShort || !(thr < INFINITY)) {
        if (lane == 0) {
          const int pos = atomicAdd(&a.st->flag2_count, 1);
          a.flags2[pos] = (int)row;
        }
        continue;
      }
      double d = INFINITY;
      int dj = 0x7fffffff;
      if (mine >= 0) {
        d = row_dist<L>(a, row, cb, mine);
        dj = mine;
        if (!(d < INFINITY)) {  // NaN / inf never wins a strict < (index 0 if nothing does)
          d = INFINITY;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, d, off);
        const int oj = __shfl_xor_sync(0xffffffffu, dj, off);
        if (od < d || (od == d && oj < dj)) {
          d = od;
          dj = oj;
        }
      }
      if (lane == 0) {
        a.idx[row] = (d < INFINITY) ? dj : 0;
        store_dist(a, row, d);
      }
    }
    return;
  }
  if ((long long)blockIdx.x * NT >= count) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sW = reinterpret_cast<float*>(smem_raw);
  float* sN = sW + TK * L;
  const int ntiles = (K + TK - 1) / TK;
  for (long long base = (long long)blockIdx.x * NT; base < count; base += (long long)gridDim.x * NT) {
    const long long i = base + threadIdx.x;
    const bool valid = i < count;
    const long long row = valid ? (long long)a.flags[i] : 0;
    const float thr = valid ? a.flag_thr[i] : -INFINITY;
    float y[L];
    {
      const float4* src = reinterpret_cast<const float4*>(a.xc + row * L);
#pragma unroll
      for (int v = 0; v < L / 4; ++v) {
        const float4 t = __ldg(src + v);
        y[4 * v + 0] = __fsub_rn(t.x, a.mu[4 * v + 0]);
        y[4 * v + 1] = __fsub_rn(t.y, a.mu[4 * v + 1]);
        y[4 * v + 2] = __fsub_rn(t.z, a.mu[4 * v + 2]);
        y[4 * v + 3] = __fsub_rn(t.w, a.mu[4 * v + 3]);
      }
    }
    int list[kShort];
    int nc = 0;
    for (int t = 0; t < ntiles; ++t) {
      const int jbase = t * TK;
      const int cnt = min(TK, K - jbase);
      if (ntiles > 1 || base == (long long)blockIdx.x * NT) {
        __syncthreads();
        const float4* gW = reinterpret_cast<const float4*>(a.w + (long long)jbase * L);
        float4* dW = reinterpret_cast<float4*>(sW);
        for (int e = threadIdx.x; e < cnt * L / 4; e += NT) dW[e] = __ldg(gW + e);
        for (int e = threadIdx.x; e < cnt; e += NT) sN[e] = __ldg(a.nrm + jbase + e);
        __syncthreads();
      }
      if (!valid) continue;
#pragma unroll 2
      for (int j = 0; j < cnt; ++j) {
        const float4* wj = reinterpret_cast<const float4*>(sW + j * L);
        float v0 = sN[j], v1 = 0.f;  // two chains
#pragma unroll
        for (int c = 0; c < L / 4; ++c) {
          const float4 w4 = wj[c];
          if (c & 1) {
            v1 = fmaf(w4.x, y[4 * c + 0], v1);
            v1 = fmaf(w4.y, y[4 * c + 1], v1);
            v1 = fmaf(w4.z, y[4 * c + 2], v1);
            v1 = fmaf(w4.w, y[4 * c + 3], v1);
          } else {
            v0 = fmaf(w4.x, y[4 * c + 0], v0);
            v0 = fmaf(w4.y, y[4 * c + 1], v0);
            v0 = fmaf(w4.z, y[4 * c + 2], v0);
            v0 = fmaf(w4.w, y[4 * c + 3], v0);
          }
        }
        if (v0 + v1 <= thr) {
          if (nc < kShort) list[nc] = jbase + j;
          ++nc;
        }
      }
    }
    if (!valid) continue;
    if (nc == 0 || nc > kShort) {
      const int pos = atomicAdd(&a.st->flag2_count, 1);
      a.flags2[pos] = (int)row;
      continue;
    }
    double best = INFINITY;
    int bj = 0;  // nothing < inf -> index 0 (_kernels.py:23-32)
    for (int c = 0; c < nc; ++c) {
      const int j = list[c];
      const double d = row_dist<L>(a, row, cb, j);
      if (d < best) {
        best = d;
        bj = j;
      }
    }
    a.idx[row] = bj;
    store_dist(a, row, best);
  }
}

bool shortlist_enabled() {
  // VQB_RERANK=full selects the full FP64 scan of every queued row (A/B)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VQB_RERANK");
    v = (e && strcmp(e, "full") == 0) ? 0 : 1;
  }
  return v == 1;
}

template <int L>
static cudaError_t launch_shortlist_L(const KernelArgs& a, int sms, cudaStream_t s) {
  using C = ShortCfg<L>;
  cudaError_t e = cudaFuncSetAttribute(shortlist_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)C::kSmem);
  if (e != cudaSuccess) return e;
  {
    cudaError_t e2 = launch_k(shortlist_kernel<L>, sms * 2, C::NT, C::kSmem, s, a);
    if (e2 != cudaSuccess) return e2;
  }
  return cudaGetLastError();
}

// the full FP64 scan on the rows the reference sees
static cudaError_t launch_exact_rows(const KernelArgs& a, int use_list, int sms, cudaStream_t s) {
  if (a.x64) return launch_exact_t<double>(a, a.x64, use_list, sms, s);
  return launch_exact_t<float>(a, a.x32, use_list, sms, s);
}

cudaError_t launch_rerank(const KernelArgs& a, int sms, cudaStream_t s) {
  if (a.xc && shortlist_enabled()) {
    cudaError_t e = a.tcb ? launch_shortlist_tc(a, sms, s) : cudaSuccess;
    if (e != cudaSuccess) return e;
    switch (a.cdim) {
      case 16: e = launch_shortlist_L<16>(a, sms, s); break;
      case 32: e = launch_shortlist_L<32>(a, sms, s); break;
      case 64: e = launch_shortlist_L<64>(a, sms, s); break;
      default: e = cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    return launch_exact_rows(a, 2, sms, s);
  }
  return launch_exact_rows(a, 1, sms, s);
}

cudaError_t launch_assign(const KernelArgs& a, bool fast, int sms, cudaStream_t s) {
  if (fast) {
    // both candidate kernels are enqueued; each reads the device-side codebook
    // size and exactly one of them runs (assign_tc for tc_kmin <= K <= tc_kmax)
    cudaError_t e;
    switch (a.cdim) {
      case 16: e = launch_fast_L<16>(a, sms, s); break;
      case 32: e = launch_fast_L<32>(a, sms, s); break;
      case 64: e = launch_fast_L<64>(a, sms, s); break;
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    if (a.small_on && small_dim(a.cdim)) {
      e = launch_small_L<16>(a, sms, s);
      if (e != cudaSuccess) return e;
    }
    if (!a.tcb) return e;
    return launch_assign_tc(a, sms, s);
  }
  return launch_exact_rows(a, 0, sms, s);
}

// ---------------------------------------------------------------------------
// epilogue: exact winner distance, distortion tiles, fixed-point cell sums
// ---------------------------------------------------------------------------

// The epilogue:
//
// td_tiles_kernel (one block per 2048-row tile): the tile's fixed-tree
// distortion partial from the per-row exact FP64 distances every assignment
// path stored (sum_inorder's role, _kernels.py:92-98, in a fixed order that
// does not depend on the grid or on the number of GPUs).
//
// sums_kernel (one persistent block per SM over a contiguous row range):
// int64 fixed-point cell sums + counts.  Integer adds commute, so the result
// is deterministic for every grid shape and GPU count.
//  * small K: half-warp-private smem tables, lanes = dims, plain adds, runs
//    of one cell summed in registers first;
//  * otherwise: a block table [dim][cell] accumulated with NATIVE 32-bit smem
//    atomics -- an exact int64 add is atomicAdd on the low word (the returned
//    old value gives the carry) plus atomicAdd on the high word -- one per
//    run of equal cells in a thread's contiguous rows.  Codebooks whose table
//    would not fit are split into chunks (gridDim.y).
// Each block writes its table to a slab; reduce_partials_kernel sums them.
// threads per sums block: 768 at L = 16 (more rows in flight: cfg2 -3 % at
// K = 1024, -12 % at K = 2), 512 for wider rows (their registers; 768 was
// +6 % at L = 64)
template <int DIM>
__host__ __device__ constexpr int sum_threads() { return DIM == 16 ? 768 : 512; }
constexpr int kEpiSmem = 224 * 1024;  // + static smem stays under the 227 KB opt-in

__host__ __device__ inline bool sums_warp_sink(int K, int dim, int nthreads) {
  // 2 half-warp tables per warp + the 32-row staging slices (double rows;
  // the 16-dimension path reads rows straight from global memory, no stage)
  const long long tables = ((long long)K * dim * 8 + K * 4 + 15) / 16 * 16 * 2 * (nthreads / 32);
  const long long stage = dim == 16 ? 0 : (long long)(nthreads / 32) * 32 * 20 * 8;
  return tables + stage <= kEpiSmem;
}
// Block-table split when K x L does not fit one table: first split the
// dimensions (each piece still reads every row once in total), then the
// cells (each cell piece re-reads X).  blockIdx.y = cell piece * ndc + dim piece.
struct SumsPlan {
  int dc, ndc;
  long long kc, nkc;
};
__host__ __device__ inline SumsPlan sums_plan(int K, int dim, int nthreads) {
  SumsPlan p;
  p.dc = dim;
  p.kc = K;
  if (!sums_warp_sink(K, dim, nthreads)) {
    while (p.dc > 8 && (long long)K * (p.dc * 8 + 4) > kEpiSmem - 64) p.dc = (p.dc / 2 + 7) / 8 * 8;
    const long long kc = (kEpiSmem - 64) / ((long long)p.dc * 8 + 4);
    p.kc = kc < K ? kc : K;
  }
  p.ndc = (dim + p.dc - 1) / p.dc;
  p.nkc = (K + p.kc - 1) / p.kc;
  return p;
}
constexpr int kWStageStride = 20;
  // staged row stride (elements), padded against bank conflicts

// exact int64 accumulation from two native 32-bit shared atomics
__device__ __forceinline__ void smem_add_i64(unsigned* lo_word, int* hi_word, long long t) {
  const unsigned lo = (unsigned)(unsigned long long)t;
  int hi = (int)(t >> 32);
  const unsigned old = atomicAdd(lo_word, lo);
  if (old + lo < old) hi += 1;  // carry out of the low word
  if (hi) atomicAdd(hi_word, hi);
}

// One block per 2048-row tile: the tile's distortion partial from the
// stored per-row distances, in a fixed order (thread t sums rows t, t+256,
// ... of the tile, then a lane butterfly, then the 8 warps in order) that
// does not depend on the grid or on the number of GPUs -- sum_inorder's role
// (_kernels.py:92-98).
// Zero the low words of the exchange buffer for cells [0, K) before this
// pass's cell sums add into them (the previous pass's apply has read them).
// The limb-RED cell sums below add straight into the exchange buffer's high
// words and counts, so those are cleared here too for cells [0, K).
__device__ __forceinline__ void zero_lo_words(const KernelArgs& a, int K) {
  const long long words = (long long)K * a.dim;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < words;
       i += (long long)gridDim.x * blockDim.x) {
    a.ex.lo()[i] = 0;
    a.ex.sums()[i] = 0;
    if (i < K) a.ex.counts()[i] = 0;
  }
}

__global__ void zero_lo_kernel(KernelArgs a, int zero_cells) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  zero_lo_words(a, zero_cells ? 1 : st->size);
}

__global__ void __launch_bounds__(256) td_tiles_kernel(KernelArgs a, int zero_lo) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  if (zero_lo) zero_lo_words(a, st->size);
  __shared__ double red[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long t = blockIdx.x;
  double v[kTdTile / 256];
#pragma unroll
  for (int r = 0; r < kTdTile / 256; ++r) {
    const long long row = t * kTdTile + (long long)r * 256 + tid;
    v[r] = row < a.n ? a.dists[row] : 0.0;
  }
  double s = 0.0;
#pragma unroll
  for (int r = 0; r < kTdTile / 256; ++r) s = __dadd_rn(s, v[r]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (tid == 0) {
    double acc = 0.0;
    for (int w = 0; w < 8; ++w) acc = __dadd_rn(acc, red[w]);
    a.ex.td()[a.tile0 + t] = __double_as_longlong(acc);
  }
}

template <typename XT, int DIM>
__device__ __forceinline__ void load_row16(const XT* __restrict__ X, long long row, int dim, int c0,
                                           bool valid, XT (&xr)[16]) {
  if (!valid) {
#pragma unroll
    for (int l = 0; l < 16; ++l) xr[l] = (XT)0;
    return;
  }
  const XT* x = X + row * dim + c0;
  if constexpr (DIM > 0 && sizeof(XT) == 4) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const float4 q = __ldg(x4 + v);
      xr[4 * v] = q.x;
      xr[4 * v + 1] = q.y;
      xr[4 * v + 2] = q.z;
      xr[4 * v + 3] = q.w;
    }
  } else if constexpr (DIM > 0) {
    const double2* x2 = reinterpret_cast<const double2*>(x);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double2 q = __ldg(x2 + v);
      xr[2 * v] = q.x;
      xr[2 * v + 1] = q.y;
    }
  } else {
    for (int l = 0; l < 16; ++l) xr[l] = (c0 + l < dim) ? x[l] : (XT)0;
  }
}

template <typename XT, int DIM>
__global__ void __launch_bounds__(sum_threads<DIM>(), 1) sums_kernel(KernelArgs a, const XT* __restrict__ X,
                                                             int zero_cells, int small_only) {
  pdl_wait();
  DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = zero_cells ? 1 : st->size;
  const int dim = DIM ? DIM : a.dim;
  // small_only: launched beside sums_red_kernel (one graph serves every
  // level); this kernel takes the passes whose codebook fits warp tables
  if (small_only && !sums_warp_sink(K, dim, sum_threads<DIM>())) return;
  if (delta_go(a, st)) return;  // the incremental branch updates the running sums instead
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) st->slabs = gridDim.x;
  const int t_lo = st->lo_shift;  // per-column shifts: a.cshift
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kSumThreads = sum_threads<DIM>();
  constexpr int kWarps = kSumThreads / 32;

  const bool warp_sink = sums_warp_sink(K, dim, kSumThreads);
  const SumsPlan plan = sums_plan(K, dim, kSumThreads);
  const int chunk = blockIdx.y;
  const long long cy = chunk / plan.ndc;
  const int dy = chunk % plan.ndc;
  if (cy >= plan.nkc) return;
  const long long c_lo = cy * plan.kc;
  const long long c_hi = (c_lo + plan.kc < K) ? c_lo + plan.kc : K;
  const int ncell = (int)(c_hi - c_lo);
  const int d_lo = dy * plan.dc;
  const int d_hi = d_lo + plan.dc < dim ? d_lo + plan.dc : dim;
  const int ndim = d_hi - d_lo;  // == dim on the warp-sink path

  extern __shared__ __align__(128) unsigned char smem_raw[];
  // warp sink: 2 x kWarps half-warp tables [ncell*dim int64 | ncell u32]
  // block sink: lo u32 [dim][ncell] | hi i32 [dim][ncell] | counts u32 [ncell]
  const long long wt_bytes = ((long long)ncell * dim * 8 + ncell * 4 + 15) / 16 * 16;
  XT* wstage = reinterpret_cast<XT*>(smem_raw + wt_bytes * 2 * kWarps);  // [warps][32][kWStageStride]
  unsigned* blo = reinterpret_cast<unsigned*>(smem_raw);
  int* bhi = reinterpret_cast<int*>(blo + (long long)ncell * ndim);
  unsigned* bcounts = reinterpret_cast<unsigned*>(bhi + (long long)ncell * ndim);
  {
    const long long zbytes = warp_sink ? wt_bytes * 2 * kWarps : (long long)ncell * ndim * 8 + ncell * 4;
    uint4* z = reinterpret_cast<uint4*>(smem_raw);
    for (long long i = tid; i < (zbytes + 15) / 16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();

  const long long n = a.n;
  const long long lo = n * blockIdx.x / gridDim.x;
  const long long hi = n * (blockIdx.x + 1) / gridDim.x;
  if (!warp_sink) {
    // Block tables, lane-sequential runs: thread t owns a contiguous slice of
    // the block's rows and keeps the running per-dimension sum of the current
    // cell in registers, flushing it (one exact int64 smem add per dimension)
    // only when the cell changes.  Rows of one cell that follow each other
    // (image blocks of smooth regions) cost one atomic per run instead of one
    // per row; with no runs it is one flush per row, as the strided path.
    const long long per = (hi - lo + kSumThreads - 1) / kSumThreads;
    const long long rb = lo + (long long)tid * per;
    const long long re = min(hi, rb + per);
    for (int c0 = d_lo; c0 < d_hi; c0 += 16) {
      const int cw = d_hi - c0 < 16 ? d_hi - c0 : 16;
      long long acc[16];
#pragma unroll
      for (int l = 0; l < 16; ++l) acc[l] = 0;
      int cur = -1;
      unsigned run = 0;
      auto flush = [&]() {
#pragma unroll
        for (int l = 0; l < 16; ++l) {
          if (l < cw) {
            const long long w = (long long)(c0 + l - d_lo) * ncell + cur;
            smem_add_i64(blo + w, bhi + w, acc[l]);
          }
          acc[l] = 0;
        }
        if (dy == 0 && c0 == d_lo) atomicAdd(bcounts + cur, run);
        run = 0;
      };
      long long row = rb;
      int cell_next = row < re ? (zero_cells ? 0 : a.idx[row]) : -1;
      for (; row < re; ++row) {
        const int cell = cell_next;
        if (row + 1 < re) cell_next = zero_cells ? 0 : a.idx[row + 1];
        const int lc = (cell >= c_lo && cell < c_hi) ? cell - (int)c_lo : -1;
        if (lc != cur) {
          if (cur >= 0) flush();
          cur = lc;
        }
        if (lc >= 0) {
          XT xr[16];
          load_row16<XT, DIM>(X, row, dim, c0, true, xr);
#pragma unroll
          for (int l = 0; l < 16; ++l)
            if (l < cw) {
              long long h, lo;
              split_fixed(xr[l], __ldg(a.cshift + c0 + l), t_lo, h, lo);  // uniform: an L1 broadcast
              acc[l] += h;
              add_lo(a, cell, c0 + l, lo);
            }
          ++run;
        }
      }
      if (cur >= 0) flush();
    }
  }
  if (warp_sink) {
    // Few cells: a private table per half-warp, lanes = dimensions, plain
    // (non-atomic) read-modify-writes.  A warp loads 32 consecutive rows
    // (lanes = rows, coalesced), stages them 16 dimensions at a time, then
    // walks them two at a time: lanes 0-15 take the even row, 16-31 the odd.
    const int half = lane >> 4, hl = lane & 15;
    long long* tab = reinterpret_cast<long long*>(smem_raw + (2 * warp + half) * wt_bytes);
    unsigned* tcount = reinterpret_cast<unsigned*>(smem_raw + (2 * warp + half) * wt_bytes +
                                                   (long long)ncell * dim * 8);
    XT* xs = wstage + warp * 32 * kWStageStride;
    if (DIM == 16) {
      // lanes = dimensions straight from global memory: half-warp h reads
      // rows base + 2p + h (64 contiguous bytes per half, one coalesced
      // 128-byte request per warp), all 16 rows' loads issued before any
      // sum; consecutive rows of one cell are summed in a register and the
      // half-warp table is touched once per run (no staging, no per-row
      // read-modify-write chain through shared memory)
      const int shl = __ldg(a.cshift + hl);
      for (long long base = lo + (long long)warp * 32; base < hi; base += (long long)kWarps * 32) {
        XT xv[16];
        int cv[16];
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const long long r = base + 2 * p + half;
          const bool ok = r < hi;
          xv[p] = ok ? __ldg(X + r * 16 + hl) : (XT)0;
          cv[p] = ok ? (zero_cells ? 0 : __ldg(a.idx + r)) : -1;
        }
        long long acc = 0, acc_lo = 0;
        int cur = -1;
        unsigned run = 0;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          if (cv[p] != cur) {  // uniform within the half-warp (one row)
            if (cur >= 0) {
              tab[(long long)cur * 16 + hl] += acc;
              add_lo(a, cur, hl, acc_lo);
              if (hl == 0) tcount[cur] += run;
            }
            cur = cv[p];
            acc = 0;
            acc_lo = 0;
            run = 0;
          }
          if (cur >= 0) {
            long long h, l2;
            split_fixed(xv[p], shl, t_lo, h, l2);
            acc += h;
            acc_lo += l2;
            ++run;
          }
        }
        if (cur >= 0) {
          tab[(long long)cur * 16 + hl] += acc;
          add_lo(a, cur, hl, acc_lo);
          if (hl == 0) tcount[cur] += run;
        }
      }
    } else
    for (long long base = lo + (long long)warp * 32; base < hi; base += (long long)kWarps * 32) {
      const long long row = base + lane;
      const bool valid = row < hi;
      const int cell = valid ? (zero_cells ? 0 : a.idx[row]) : -1;
      const int lc = (valid && cell >= c_lo && cell < c_hi) ? cell - (int)c_lo : -1;
      for (int c0 = 0; c0 < dim; c0 += 16) {
        XT xr[16];
        load_row16<XT, DIM>(X, row, dim, c0, lc >= 0, xr);
#pragma unroll
        for (int l = 0; l < 16; ++l) xs[lane * kWStageStride + l] = xr[l];
        __syncwarp();
#pragma unroll 4
        for (int p = 0; p < 16; ++p) {
          const int rr = 2 * p + half;
          const int cl = __shfl_sync(0xffffffffu, lc, rr);
          if (cl >= 0) {
            if (c0 + hl < dim) {
              long long h, l2;
              split_fixed(xs[rr * kWStageStride + hl], __ldg(a.cshift + c0 + hl), t_lo, h, l2);
              tab[(long long)cl * dim + c0 + hl] += h;
              add_lo(a, cl, c0 + hl, l2);
            }
            if (c0 == 0 && hl == 0) tcount[cl] += 1;
          }
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // block slab [blockIdx.x][K*dim sums | K counts] (int64)
  long long* slab = a.partials + (long long)blockIdx.x * ((long long)a.kmax * dim + a.kmax);
  const long long words = (long long)ncell * dim;
  if (warp_sink) {
    for (long long i = tid; i < words; i += blockDim.x) {
      long long v = 0;
      for (int w = 0; w < 2 * kWarps; ++w) v += reinterpret_cast<const long long*>(smem_raw + w * wt_bytes)[i];
      slab[c_lo * dim + i] = v;
    }
    for (int i = tid; i < ncell; i += blockDim.x) {
      long long v = 0;
      for (int w = 0; w < 2 * kWarps; ++w)
        v += reinterpret_cast<const unsigned*>(smem_raw + w * wt_bytes + words * 8)[i];
      slab[(long long)K * dim + c_lo + i] = v;
    }
  } else {
    for (long long i = tid; i < (long long)ncell * ndim; i += blockDim.x) {
      const long long cl = i / ndim, l = i % ndim;
      const long long w = l * ncell + cl;
      slab[(c_lo + cl) * dim + d_lo + l] = (long long)(((unsigned long long)(unsigned)bhi[w] << 32) + blo[w]);
    }
    if (dy == 0)
      for (int i = tid; i < ncell; i += blockDim.x) slab[(long long)K * dim + c_lo + i] = bcounts[i];
  }
}

// ---------------------------------------------------------------------------
// Cell sums for larger codebooks without returning atomics ("limb REDs").
//
// A coordinate's high word h (|h| < 2^(t-1), t = lo_shift = 62 - e_n) is
// biased to u = h + 2^(t-1) in [0, 2^t) and cut into m limbs of w bits; each
// limb is added to a 32-bit shared-memory counter with a NON-returning RED
// (one ATOMS.ADD, no carry to wait for).  A counter absorbs 2^(32-w) adds, and
// w is chosen so that exceeds the rows one CTA visits, so no limb can wrap.
// At the end the CTA recombines sum_j limb_j 2^(w j) - count * 2^(t-1) --
// exactly its share of the cell sum -- and adds it into the exchange buffer
// with one 64-bit global atomic per (cell, dim) (integer adds commute: the
// result does not depend on the order).  Codebooks too large for a table of
// all dims are split into dimension pieces (blockIdx.x % pieces, adjacent in
// launch order so the pieces of one row chunk share its rows through L2).
// ---------------------------------------------------------------------------
struct LimbPlan {
  int m, w;         // limbs per coordinate, bits per limb
  int lp, pieces;   // dims per piece (template LP), pieces
  int chunks;       // row chunks
  long long rows;   // rows per chunk
  int small_cut;    // codebooks up to this size are left to sums_kernel's warp tables (0: none)
};
__host__ __device__ inline LimbPlan limb_plan(long long n, int K, int dim, int lo_shift, int sms) {
  LimbPlan p{};
  const int t = lo_shift;
  // dims per piece: the widest of 32 / 16 / 8 / 4 whose table fits
  const long long budget = kEpiSmem - 1024;
  int lp = 32;
  while (lp > 4 && (long long)K * (lp * 4 * 3 + 4) > budget) lp >>= 1;
  if (lp > 16 && dim <= 16) lp = 16;
  p.lp = lp;
  p.pieces = (dim + lp - 1) / lp;
  p.chunks = sms / p.pieces > 0 ? sms / p.pieces : 1;
  if ((long long)p.chunks * 4096 > n) p.chunks = (int)((n + 4095) / 4096) > 0 ? (int)((n + 4095) / 4096) : 1;
  p.rows = (n + p.chunks - 1) / p.chunks;
  int hb = 0;
  while (hb < 40 && (1LL << hb) <= p.rows) ++hb;  // rows < 2^hb
  p.w = 32 - hb;                                     // 2^(32-w) = 2^hb > rows
  if (p.w > 31) p.w = 31;
  p.m = p.w > 0 ? (t + p.w - 1) / p.w : 99;
  return p;
}
__host__ __device__ inline bool limb_ok(const LimbPlan& p, int K) {
  return p.w >= 8 && p.m <= 4 && (long long)K * (p.lp * 4 * p.m + 4) <= kEpiSmem - 1024;
}

// 4 consecutive coordinates of a row (one 16-byte load for float rows)
template <typename XT>
__device__ __forceinline__ void load4(const XT* __restrict__ p, int valid, bool vec, XT (&v)[4]) {
  if (valid == 4 && vec) {
    if constexpr (sizeof(XT) == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      const double2 q0 = __ldg(reinterpret_cast<const double2*>(p));
      const double2 q1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
      v[0] = q0.x; v[1] = q0.y; v[2] = q1.x; v[3] = q1.y;
    }
  } else {
#pragma unroll
    for (int g = 0; g < 4; ++g) v[g] = g < valid ? __ldg(p + g) : (XT)0;
  }
}

// incremental branch inside sums_red_kernel (1) or as its own launch (0).
// Merged it saves one idle launch per pass (design -1 %), but the larger
// kernel's full-sum path ran 12-15 us slower at cfg2 / cfg3 (the stateless
// Lloyd step: +4 %), so it is its own launch.
#ifndef VQB_DELTA_MERGE
#define VQB_DELTA_MERGE 0
#endif
template <typename XT, int LP, int M>
__device__ __forceinline__ void sums_delta_body(const KernelArgs& a, const XT* __restrict__ X, const LimbPlan& pl);

template <typename XT, int LP, int M>
__global__ void __launch_bounds__(512, 1) sums_red_kernel(KernelArgs a, const XT* __restrict__ X, int zero_cells,
                                                          LimbPlan pl) {
  pdl_wait();
  DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = zero_cells ? 1 : st->size;
  const int dim = a.dim;
#if VQB_DELTA_MERGE
  if (delta_go(a, st)) {  // the incremental pass: only the rows that changed cell (same tables, same plan)
    sums_delta_body<XT, LP, M>(a, X, pl);
    return;
  }
#else
  if (delta_go(a, st)) return;
#endif
  if (pl.small_cut > 0 && K <= pl.small_cut) return;  // sums_kernel's warp tables take this pass
  if (blockIdx.x == 0 && threadIdx.x == 0) st->slabs = pl.chunks;
  const int t = st->lo_shift;  // == fixed_lo_shift(n_global), what the plan was made for
  constexpr int m = M;
  const int w = pl.w;
  const int piece = blockIdx.x % pl.pieces;
  const long long chunk = blockIdx.x / pl.pieces;
  const int d0 = piece * LP;
  constexpr int TPR = LP / 4;  // threads per row: 4 coordinates each
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // one record per cell: LP x m limb counters + the row count.  The record
  // length is odd, so the records of the random cells a warp touches spread
  // over all 32 banks (LP x m alone is a multiple of 4: a quarter of them)
  constexpr int kRec = LP * M + 1;
  unsigned* tab = reinterpret_cast<unsigned*>(smem_raw);     // [K][LP x m | count]
  const long long twords = (long long)K * kRec;
  for (long long i = threadIdx.x; i < twords; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  const long long r0 = chunk * pl.rows;
  const long long r1 = r0 + pl.rows < a.n ? r0 + pl.rows : a.n;
  const int g0 = (threadIdx.x % TPR) * 4;  // first of this thread's 4 dims within the piece
  const int d = d0 + g0;
  const int valid = dim - d >= 4 ? 4 : (dim - d > 0 ? dim - d : 0);
  const bool vec = (dim & 3) == 0;  // 16-byte aligned row slices
  int sh[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) sh[g] = g < valid ? __ldg(a.cshift + d + g) : 0;
  const long long bias = 1LL << (t - 1);
  const unsigned long long mask = (1ull << w) - 1;
  const int rstep = blockDim.x / TPR;
  constexpr int U = sizeof(XT) == 4 ? 8 : 4;  // rows per thread per batch; the next batch is in flight meanwhile
  // dims past `dim` load as 0 and add into table entries the flush skips
  XT xv[U][4];
  int cv[U];
  auto fetch = [&](long long rb) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long row = rb + (long long)u * rstep;
      const bool ok = row < r1;
      cv[u] = ok ? (zero_cells ? 0 : __ldg(a.idx + row)) : -1;
      load4<XT>(X + row * dim + d, ok ? valid : 0, vec, xv[u]);
    }
  };
  long long rb = r0 + threadIdx.x / TPR;
  if (rb < r1) fetch(rb);
  while (rb < r1) {
    XT cx[U][4];
    int cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cc[u] = cv[u];
#pragma unroll
      for (int g = 0; g < 4; ++g) cx[u][g] = xv[u][g];
    }
    const long long nb = rb + (long long)rstep * U;
    if (nb < r1) fetch(nb);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = cc[u];
      if (c < 0) continue;
      if (g0 == 0) atomicAdd(tab + (unsigned)c * (unsigned)kRec + (unsigned)(LP * M), 1u);
      unsigned* e = tab + (unsigned)c * (unsigned)kRec + (unsigned)(g0 * M);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        long long h;
        if (!split_fast(cx[u][g], sh[g], h)) {  // rare for float32 rows: bits below the grid
          long long lo;
          split_fixed(cx[u][g], sh[g], t, h, lo);
          add_lo(a, c, d + g, lo);
        }
        const unsigned long long uv = (unsigned long long)(h + bias);
#pragma unroll
        for (int j = 0; j < M; ++j) atomicAdd(e + g * M + j, (unsigned)((uv >> (w * j)) & mask));
      }
    }
    rb = nb;
  }
  __syncthreads();
  // this chunk's share of the sums into its slab (reduce_partials_kernel adds
  // the slabs in a fixed order; every word of cells < K is written)
  long long* slab = a.partials + chunk * ((long long)a.kmax * dim + a.kmax);
  for (long long i = threadIdx.x; i < (long long)K * LP; i += blockDim.x) {
    const long long c = i / LP;
    const int ll = (int)(i % LP);
    if (d0 + ll >= dim) continue;
    const unsigned* e = tab + c * kRec + ll * m;
    long long v = 0;
    for (int j = 0; j < m; ++j) v += (long long)e[j] << (w * j);
    slab[c * dim + d0 + ll] = v - (long long)tab[c * kRec + LP * M] * bias;
  }
  if (piece == 0)
    for (long long c = threadIdx.x; c < K; c += blockDim.x) slab[(long long)K * dim + c] = tab[c * kRec + LP * M];
}

// Launch the limb-RED sums when the plan fits (K large enough that the
// warp-private tables are out, small enough that a table of >= 4 dims fits);
// *used tells the caller whether the slab reduction is still needed.
template <typename XT, int LP, int M>
static cudaError_t launch_red_lpm(const KernelArgs& a, const XT* X, const LimbPlan& pl, bool zero_cells,
                                  cudaStream_t s) {
  const size_t smem = (size_t)a.kmax * (LP * M + 1) * 4;
  cudaError_t e = cudaFuncSetAttribute(sums_red_kernel<XT, LP, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  return launch_k(sums_red_kernel<XT, LP, M>, (unsigned)(pl.chunks * pl.pieces), 512, smem, s, a, X,
                  zero_cells ? 1 : 0, pl);
}
template <typename XT, int LP>
static cudaError_t launch_red_lp(const KernelArgs& a, const XT* X, const LimbPlan& pl, bool zero_cells,
                                 cudaStream_t s) {
  switch (pl.m) {
    case 2: return launch_red_lpm<XT, LP, 2>(a, X, pl, zero_cells, s);
    case 3: return launch_red_lpm<XT, LP, 3>(a, X, pl, zero_cells, s);
    default: return launch_red_lpm<XT, LP, 4>(a, X, pl, zero_cells, s);
  }
}

template <typename XT>
static cudaError_t launch_sums_red(const KernelArgs& a, const XT* X, bool zero_cells, int sms, cudaStream_t s,
                                   bool* used, int* chunks, int small_cut) {
  *used = false;
  if (zero_cells) return cudaSuccess;
  LimbPlan pl = limb_plan(a.n, (int)a.kmax, a.dim, fixed_lo_shift(a.n_global), sms);
  pl.small_cut = small_cut;
  if (!limb_ok(pl, (int)a.kmax)) return cudaSuccess;
  *used = true;
  *chunks = pl.chunks;
  switch (pl.lp) {
    case 32: return launch_red_lp<XT, 32>(a, X, pl, zero_cells, s);
    case 16: return launch_red_lp<XT, 16>(a, X, pl, zero_cells, s);
    case 8: return launch_red_lp<XT, 8>(a, X, pl, zero_cells, s);
    default: return launch_red_lp<XT, 4>(a, X, pl, zero_cells, s);
  }
}

// ---------------------------------------------------------------------------
// Incremental cell sums of the training loop (vqb200_internal.h delta_go).
// moved_scan_kernel compares the pass's cells with the previous pass's, lists
// the rows that changed cell and brings idx_prev up to date; sums_delta_kernel
// adds each listed row into its new cell and takes it out of its old one in
// the limb tables of sums_red_kernel (a removal adds the negated limbs: the
// 32-bit counters are read back as signed, so a CTA flushes before either
// side of a counter can reach 2^31); reduce_partials_kernel adds the slabs to
// the running sums `acc` and publishes them in the exchange buffer -- or,
// after a pass that summed every row, keeps that pass's local sums as the new
// running sums.  Reference: _kernels.update_rows (_kernels.py:39-66)
// computes the same sums from scratch every pass.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) moved_scan_kernel(KernelArgs a) {
  pdl_wait();
  DevState* st = a.st;
  if (pass_off(st) || !delta_track(a, st)) return;
  const bool list = st->acc_size == st->size;  // else: this pass sums every row; only idx_prev is refreshed
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int wtot[kScanThreads / 32];
  __shared__ int bbase;
  const long long items = (a.n + 3) / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // whole blocks iterate (the list positions of a block's rows come from one
  // global atomic per block and iteration)
  for (long long b0 = (long long)blockIdx.x * blockDim.x; b0 < items; b0 += stride) {
    const long long i = b0 + threadIdx.x;
    int cur[4] = {0, 0, 0, 0}, prv[4] = {0, 0, 0, 0};
    unsigned m = 0;
    if (i < items) {
      const long long r = 4 * i;
      if (r + 3 < a.n) {
        const int4 c = *reinterpret_cast<const int4*>(a.idx + r);
        const int4 q = *reinterpret_cast<const int4*>(a.idx_prev + r);
        cur[0] = c.x; cur[1] = c.y; cur[2] = c.z; cur[3] = c.w;
        prv[0] = q.x; prv[1] = q.y; prv[2] = q.z; prv[3] = q.w;
      } else {
        for (int k = 0; k < 4; ++k)
          if (r + k < a.n) {
            cur[k] = a.idx[r + k];
            prv[k] = a.idx_prev[r + k];
          }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) m |= (cur[k] != prv[k]) ? (1u << k) : 0u;
      if (m) {
        if (r + 3 < a.n) {
          *reinterpret_cast<int4*>(a.idx_prev + r) = make_int4(cur[0], cur[1], cur[2], cur[3]);
        } else {
          for (int k = 0; k < 4; ++k)
            if (r + k < a.n) a.idx_prev[r + k] = cur[k];
        }
      }
    }
    if (!list) continue;  // uniform over the grid
    const int cnt = __popc(m);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int t = wtot[lane];
      int ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += v;
      }
      wtot[lane] = ti - t;  // exclusive warp offsets
      if (lane == 31) bbase = ti > 0 ? atomicAdd(&st->nmoved, ti) : 0;
    }
    __syncthreads();
    long long pos = (long long)bbase + wtot[warp] + incl - cnt;
    __syncthreads();  // wtot / bbase are rewritten by the next iteration
    // past delta_max the pass sums every row anyway: the list is not read
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if ((m >> k) & 1u) {
        if (pos < a.mv_cap) {
          a.mv[pos] = (int)(4 * i + k);
          a.mv[a.mv_cap + pos] = prv[k];
          a.mv[2 * a.mv_cap + pos] = cur[k];
        }
        ++pos;
      }
  }
}

__device__ __forceinline__ void add_lo_acc(const KernelArgs& a, long long cell, int l, long long lo) {
  long long* acc_lo = a.acc + a.kmax * a.dim + a.kmax;
  if (lo) atomicAdd(reinterpret_cast<unsigned long long*>(acc_lo + cell * a.dim + l), (unsigned long long)lo);
}

constexpr long long kDeltaMinEntries = 1024;  // listed rows per CTA before another CTA (and slab) joins
template <typename XT, int LP, int M>
__device__ __forceinline__ void sums_delta_body(const KernelArgs& a, const XT* __restrict__ X, const LimbPlan& pl) {
  DevState* st = a.st;
  const long long nm = st->nmoved;
  if (nm == 0) return;  // the slab reduction republishes the running sums
  const int K = st->size;
  const int dim = a.dim;
  // few listed rows: few CTAs (and slabs to reduce afterwards)
  long long used = (nm + kDeltaMinEntries - 1) / kDeltaMinEntries;
  used = used < pl.chunks ? used : pl.chunks;
  if (blockIdx.x / pl.pieces >= used) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->slabs = (int)used;
  const int t = st->lo_shift;
  constexpr int m = M;
  const int w = pl.w;
  const int piece = blockIdx.x % pl.pieces;
  const long long chunk = blockIdx.x / pl.pieces;
  const int d0 = piece * LP;
  constexpr int TPR = LP / 4;
  constexpr int kRec = LP * M + 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned* tab = reinterpret_cast<unsigned*>(smem_raw);  // [K][LP x m | count], signed mod 2^32
  const long long twords = (long long)K * kRec;
  const long long per = (nm + used - 1) / used;
  const long long e0 = chunk * per;
  const long long e1 = e0 + per < nm ? e0 + per : nm;
  // a counter takes at most one limb (< 2^w) per entry on either side
  const long long round = 1LL << (31 - w);
  const int g0 = (threadIdx.x % TPR) * 4;
  const int d = d0 + g0;
  const int valid = dim - d >= 4 ? 4 : (dim - d > 0 ? dim - d : 0);
  const bool vec = (dim & 3) == 0;
  int sh[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) sh[g] = g < valid ? __ldg(a.cshift + d + g) : 0;
  const long long bias = 1LL << (t - 1);
  const unsigned long long mask = (1ull << w) - 1;
  const int rstep = blockDim.x / TPR;
  constexpr int U = 4;  // entries per thread per batch; the next batch is in flight meanwhile
  long long* slab = a.partials + chunk * ((long long)a.kmax * dim + a.kmax);
  bool first = true;
  for (long long s0 = e0; first || s0 < e1; s0 += round) {
    for (long long i = threadIdx.x; i < twords; i += blockDim.x) tab[i] = 0;
    __syncthreads();
    const long long s1 = s0 + round < e1 ? s0 + round : e1;
    XT xv[U][4];
    int cn[U], co[U];
    auto fetch = [&](long long eb) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long e = eb + (long long)u * rstep;
        const bool ok = e < s1;
        const long long row = ok ? (long long)__ldg(a.mv + e) : 0;
        co[u] = ok ? __ldg(a.mv + a.mv_cap + e) : -1;
        cn[u] = ok ? __ldg(a.mv + 2 * a.mv_cap + e) : -1;
        load4<XT>(X + row * dim + d, ok ? valid : 0, vec, xv[u]);
      }
    };
    long long eb = s0 + threadIdx.x / TPR;
    if (eb < s1) fetch(eb);
    while (eb < s1) {
      XT cx[U][4];
      int ccn[U], cco[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ccn[u] = cn[u];
        cco[u] = co[u];
#pragma unroll
        for (int g = 0; g < 4; ++g) cx[u][g] = xv[u][g];
      }
      const long long nb = eb + (long long)rstep * U;
      if (nb < s1) fetch(nb);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (ccn[u] < 0) continue;
        unsigned* en = tab + (unsigned)ccn[u] * (unsigned)kRec;
        unsigned* eo = tab + (unsigned)cco[u] * (unsigned)kRec;
        if (g0 == 0) {
          atomicAdd(en + LP * M, 1u);
          atomicAdd(eo + LP * M, 0xffffffffu);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          long long h;
          if (!split_fast(cx[u][g], sh[g], h)) {
            long long lo;
            split_fixed(cx[u][g], sh[g], t, h, lo);
            if (g < valid) {
              add_lo_acc(a, ccn[u], d + g, lo);
              add_lo_acc(a, cco[u], d + g, -lo);
            }
          }
          const unsigned long long uv = (unsigned long long)(h + bias);
#pragma unroll
          for (int j = 0; j < M; ++j) {
            const unsigned limb = (unsigned)((uv >> (w * j)) & mask);
            atomicAdd(en + (g0 + g) * M + j, limb);
            atomicAdd(eo + (g0 + g) * M + j, 0u - limb);
          }
        }
      }
      eb = nb;
    }
    __syncthreads();
    // signed limb sums -> this chunk's slab (every word of cells < K written)
    for (long long i = threadIdx.x; i < (long long)K * LP; i += blockDim.x) {
      const long long c = i / LP;
      const int ll = (int)(i % LP);
      if (d0 + ll >= dim) continue;
      const unsigned* e = tab + c * kRec + ll * m;
      long long v = 0;
      for (int j = 0; j < m; ++j) v += (long long)(int)e[j] << (w * j);
      v -= (long long)(int)tab[c * kRec + LP * M] * bias;
      long long* dst = slab + c * dim + d0 + ll;
      *dst = first ? v : *dst + v;
    }
    if (piece == 0)
      for (long long c = threadIdx.x; c < K; c += blockDim.x) {
        long long* dst = slab + (long long)K * dim + c;
        const long long v = (long long)(int)tab[c * kRec + LP * M];
        *dst = first ? v : *dst + v;
      }
    __syncthreads();
    first = false;
  }
}

// the incremental sums as their own launch (codebooks whose every level fits
// the warp tables have no sums_red_kernel in their pass; otherwise that
// kernel takes the incremental branch itself)
template <typename XT, int LP, int M>
__global__ void __launch_bounds__(512, 1) sums_delta_kernel(KernelArgs a, const XT* __restrict__ X, LimbPlan pl) {
  pdl_wait();
  if (pass_off(a.st) || !delta_go(a, a.st)) return;
  sums_delta_body<XT, LP, M>(a, X, pl);
}

template <typename XT, int LP>
static cudaError_t launch_delta_lp(const KernelArgs& a, const XT* X, const LimbPlan& pl, cudaStream_t s) {
  const unsigned grid = (unsigned)(pl.chunks * pl.pieces);
#define VQB_DELTA_M(MM)                                                                                      \
  {                                                                                                          \
    const size_t smem = (size_t)a.kmax * (LP * MM + 1) * 4;                                                  \
    cudaError_t e = cudaFuncSetAttribute(sums_delta_kernel<XT, LP, MM>,                                      \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);            \
    if (e != cudaSuccess) return e;                                                                          \
    return launch_k(sums_delta_kernel<XT, LP, MM>, grid, 512, smem, s, a, X, pl);                            \
  }
  switch (pl.m) {
    case 2: VQB_DELTA_M(2)
    case 3: VQB_DELTA_M(3)
    default: VQB_DELTA_M(4)
  }
#undef VQB_DELTA_M
}

// the incremental sums' own launch, for passes without a sums_red_kernel
template <typename XT>
static cudaError_t launch_delta(const KernelArgs& a, const XT* X, const LimbPlan& pl, cudaStream_t s) {
  switch (pl.lp) {
    case 32: return launch_delta_lp<XT, 32>(a, X, pl, s);
    case 16: return launch_delta_lp<XT, 16>(a, X, pl, s);
    case 8: return launch_delta_lp<XT, 8>(a, X, pl, s);
    default: return launch_delta_lp<XT, 4>(a, X, pl, s);
  }
}

// sum the per-block slabs into the exchange buffer: 32 words x 8 slab groups
// per 256-thread block, int64 (any order is exact)
// Incremental passes (delta_go): the slabs hold the moved rows' signed
// contributions -- added to the running sums `acc`, which are then published;
// a training pass that summed every row leaves its local sums in `acc`.
__global__ void __launch_bounds__(256) reduce_partials_kernel(KernelArgs a, int nblocks, int zero_cells) {
  pdl_wait();
  const DevState* st = a.st;
  if (pass_off(st)) return;
  const bool track = !zero_cells && delta_track(a, st);
  const bool go = track && delta_go(a, st);
  if (go)
    nblocks = st->nmoved > 0 ? st->slabs : 0;
  else if (nblocks < 0)
    nblocks = st->slabs;  // whichever sums kernel ran this pass
  const int K = zero_cells ? 1 : st->size;
  const long long dim = a.dim;
  const long long words = (long long)K * dim + K;
  const long long stride = a.kmax * dim + a.kmax;
  long long* acc_c = a.acc + a.kmax * dim;
  long long* acc_l = acc_c + a.kmax;
  __shared__ long long part[8][32];
  const int wl = threadIdx.x & 31, g = threadIdx.x >> 5;
  for (long long w0 = (long long)blockIdx.x * 32; w0 < words; w0 += (long long)gridDim.x * 32) {
    const long long w = w0 + wl;
    long long v0 = 0, v1 = 0, v2 = 0, v3 = 0;
    if (w < words) {
      int b = g;
      for (; b + 24 < nblocks; b += 32) {
        v0 += a.partials[(long long)b * stride + w];
        v1 += a.partials[(long long)(b + 8) * stride + w];
        v2 += a.partials[(long long)(b + 16) * stride + w];
        v3 += a.partials[(long long)(b + 24) * stride + w];
      }
      for (; b < nblocks; b += 8) v0 += a.partials[(long long)b * stride + w];
    }
    part[g][wl] = v0 + v1 + v2 + v3;
    __syncthreads();
    if (g == 0 && w < words) {
      long long v = 0;
      for (int k = 0; k < 8; ++k) v += part[k][wl];
      const bool is_sum = w < K * dim;
      long long* accw = is_sum ? a.acc + w : acc_c + (w - K * dim);
      if (go) v += *accw;
      if (is_sum)
        a.ex.sums()[w] = v;
      else
        a.ex.counts()[w - K * dim] = v;
      if (track) {
        *accw = v;
        if (is_sum) {
          if (go)
            a.ex.lo()[w] = acc_l[w];
          else
            acc_l[w] = a.ex.lo()[w];
        }
      }
    }
    __syncthreads();
  }
}

template <typename XT, int DIM>
static cudaError_t launch_full_sums(const KernelArgs& a, const XT* X, bool zero_cells, int sms, cudaStream_t s,
                                    const LimbPlan& dpl);

template <typename XT, int DIM>
static cudaError_t launch_epi_dim(const KernelArgs& a_in, const XT* X, bool want_td, bool want_sums,
                                  bool zero_cells, int sms, cudaStream_t s) {
  cudaError_t e;
  KernelArgs a = a_in;
  // incremental sums: only where the limb tables of the largest codebook fit
  LimbPlan dpl{};
  if (a.acc) {
    dpl = limb_plan(a.n, (int)a.kmax, a.dim, fixed_lo_shift(a.n_global), sms);
    if (!want_sums || zero_cells || !limb_ok(dpl, (int)a.kmax)) a.acc = nullptr;
  }
  if (want_td && !zero_cells) {
    // every assignment path stored the rows' exact distances (store_dist);
    // the same grid clears the low words the cell sums below add into
    const long long ntiles = (a.n + kTdTile - 1) / kTdTile;
    e = launch_k(td_tiles_kernel, (unsigned)ntiles, 256, 0, s, a, want_sums ? 1 : 0);
    if (e != cudaSuccess) return e;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  } else if (want_sums) {
    e = launch_k(zero_lo_kernel, 64, 256, 0, s, a, zero_cells ? 1 : 0);
    if (e != cudaSuccess) return e;
  }
  if (!want_sums) return cudaSuccess;
  if (a.acc) {
    e = launch_k(moved_scan_kernel, sms * 2, kScanThreads, 0, s, a);
    if (e != cudaSuccess) return e;
  }
  return launch_full_sums<XT, DIM>(a, X, zero_cells, sms, s, dpl);
}

// The sums kernels of a pass and the slab reduction.  Each reads the pass's
// codebook size and mode from the device state and exactly one does the work:
// sums_kernel (warp tables, small codebooks), sums_red_kernel (limb REDs; on
// incremental passes its sums_delta branch) or, where a design has no
// sums_red_kernel, sums_delta_kernel.
template <typename XT, int DIM>
static cudaError_t launch_full_sums(const KernelArgs& a, const XT* X, bool zero_cells, int sms, cudaStream_t s,
                                    const LimbPlan& dpl) {
  cudaError_t e;
  const long long kmax = zero_cells ? 1 : a.kmax;
  constexpr int kSumThreads = sum_threads<DIM>();
  const long long words = kmax * a.dim + kmax;
  int rb = (int)((words + 31) / 32);
  if (rb > 8192) rb = 8192;
  const int red_mode = getenv_flag("VQB_SUMS_RED", 1);  // 0 never, 1 for codebooks past the warp tables
  const long long rows_per_block = 4LL * kSumThreads;
  int blocks = (int)((a.n + rows_per_block - 1) / rows_per_block);
  if (blocks > sms) blocks = sms;
  if (blocks < 1) blocks = 1;
  e = cudaFuncSetAttribute(sums_kernel<XT, DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEpiSmem);
  if (e != cudaSuccess) return e;
  if (!zero_cells && red_mode == 1 && !sums_warp_sink((int)kmax, a.dim, kSumThreads)) {
    // one graph serves every level: the warp-table kernel takes the small
    // codebooks (no shared-address contention), the limb-RED kernel the rest
    bool used = false;
    int chunks = 0;
    int cut = 0;
    while (cut < kmax && sums_warp_sink(cut + 1, a.dim, kSumThreads)) ++cut;
    e = launch_sums_red<XT>(a, X, zero_cells, sms, s, &used, &chunks, cut);
    if (e != cudaSuccess) return e;
    if (used) {
      if (cut > 0) {
        const SumsPlan p1 = sums_plan(cut, a.dim, kSumThreads);
        e = launch_k(sums_kernel<XT, DIM>, dim3(blocks, (unsigned)(p1.nkc * p1.ndc)), kSumThreads, kEpiSmem, s, a,
                     X, 0, 1);
        if (e != cudaSuccess) return e;
      }
#if !VQB_DELTA_MERGE
      if (a.acc) {
        e = launch_delta<XT>(a, X, dpl, s);
        if (e != cudaSuccess) return e;
      }
#endif
      return launch_k(reduce_partials_kernel, rb, 256, 0, s, a, -1, 0);
    }
  }
  const SumsPlan plan = sums_plan((int)kmax, a.dim, kSumThreads);
  const int chunks = (int)(plan.nkc * plan.ndc);
  e = launch_k(sums_kernel<XT, DIM>, dim3(blocks, chunks), kSumThreads, kEpiSmem, s, a, X, zero_cells ? 1 : 0, 0);
  if (e != cudaSuccess) return e;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (a.acc) {
    e = launch_delta<XT>(a, X, dpl, s);
    if (e != cudaSuccess) return e;
  }
  e = launch_k(reduce_partials_kernel, rb, 256, 0, s, a, blocks, zero_cells ? 1 : 0);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <typename XT>
static cudaError_t launch_epi_t(const KernelArgs& a, const XT* X, bool want_dists, bool want_sums,
                                bool zero_cells, int sms, cudaStream_t s) {

  switch (a.dim) {
    case 16: return launch_epi_dim<XT, 16>(a, X, want_dists, want_sums, zero_cells, sms, s);
    case 32: return launch_epi_dim<XT, 32>(a, X, want_dists, want_sums, zero_cells, sms, s);
    case 64: return launch_epi_dim<XT, 64>(a, X, want_dists, want_sums, zero_cells, sms, s);
    default: return launch_epi_dim<XT, 0>(a, X, want_dists, want_sums, zero_cells, sms, s);
  }
}

cudaError_t launch_epilogue(const KernelArgs& a, bool want_dists, bool want_sums, bool zero_cells,
                            int sms, cudaStream_t s) {
  if (a.x32) return launch_epi_t<float>(a, a.x32, want_dists, want_sums, zero_cells, sms, s);
  return launch_epi_t<double>(a, a.x64, want_dists, want_sums, zero_cells, sms, s);
}

// ---------------------------------------------------------------------------
// finalize (one block): the pass's distortion, the convergence test
// (core.py:342-356), level / guard logic (core.py:384-415) and history.  It
// only DECIDES: the codebook work (centroids, split, FP32 staging) is done
// by apply_kernel over all SMs.  phase 0 = after the initial column-sum pass.
// ---------------------------------------------------------------------------

__device__ void record_hist(DevState* st, int size, int it, double td, long long empty) {
  {
    HistRec& h = st->hist[st->n_hist % st->hist_cap];  // ring: the host drains it per batch
    h.size = size;
    h.iteration = it;
    h.td = td;
    h.empty = empty;
    h.t_ns = globaltimer();
  }
  st->n_hist += 1;
}

// action bits for apply_kernel
constexpr int kActUpdate = 1;
constexpr int kActSplit = 2;

__device__ __forceinline__ void set_action(DevState* st, int act) {
  // the source codebook is the current one; the result goes to the other buffer
  st->act = act;
  st->act_src = st->cur;
  st->act_k = st->size;
  st->cur ^= 1;
  if (act & kActSplit) {
    st->size = 2 * st->size;
    st->iteration = 1;
    st->td_prev = INFINITY;
  }
}

// The decision step of a pass, one block of any size (<= 1024 threads).
__device__ void finalize_body(const KernelArgs& a, int phase, bool track = true) {
  DevState* st = a.st;
  __shared__ double red[32];
  __shared__ long long s_empty[32];
  __shared__ double s_td;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    st->tc_bad = 0;  // apply_kernel re-stages the operand image
    st->flagged_total += st->flag_count;
    st->flagged2_total += st->flag2_count;
    st->flag_count = 0;
    st->flag2_count = 0;
  }

  if (phase == 0) {
    // global centroid = column sums / m (core.py:380, parallel.py:273): an
    // "update" of the size-1 codebook whose single cell holds every row,
    // followed by the first split unless target_size == 1 (core.py:417-422)
    if (tid == 0) {
      st->t0_ns = globaltimer();
      if (st->target <= 1) {
        st->mode = kModeFinalAssign;
        set_action(st, kActUpdate);
      } else {
        set_action(st, kActUpdate | kActSplit);
      }
    }
    return;
  }

  // ---- distortion of this pass (fixed tree over tiles; in-order if ordered)
  const int K = st->size;
  if (tid == 0) {
    // the running sums / previous cells now describe this codebook size (the
    // fused pass keeps neither)
    st->acc_size = track && delta_track(a, st) ? K : 0;
    st->nmoved = 0;
  }
  if (st->mode != kModeUpdateOnly) {
    if (st->ordered) {
      if (tid == 0) {
        double s = 0.0;  // _kernels.sum_inorder (_kernels.py:92-98)
        for (long long i = 0; i < a.n; ++i) s = __dadd_rn(s, a.dists[i]);
        s_td = s;
      }
    } else {
      // a fixed tree of 256 leaves whatever the block size (the fused pass
      // runs this with 512 threads: its extra warps add exact zeros), so the
      // distortion has the same bits on every path
      const long long nt = a.ex.ntiles;
      const long long per = (nt + 255) / 256;
      double s = 0.0;
      if (tid < 256)
        for (long long i = tid * per; i < (tid + 1) * per && i < nt; ++i)
          s = __dadd_rn(s, __longlong_as_double(a.ex.td()[i]));
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
      if (lane == 0) red[warp] = s;
      __syncthreads();
      if (tid == 0) {
        double t2 = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t2 = __dadd_rn(t2, red[w]);
        s_td = t2;
      }
    }
  }
  // ---- empty cells (counts == 0) of this pass
  long long e = 0;
  for (int k = tid; k < K; k += blockDim.x) e += (a.ex.counts()[k] == 0);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
  if (lane == 0) s_empty[warp] = e;
  __syncthreads();
  if (tid != 0) return;
  long long empties = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) empties += s_empty[w];
  const double td = s_td;

  if (st->mode == kModeUpdateOnly) {
    st->last_empty = empties;
    set_action(st, kActUpdate);
    st->done = 1;
    return;
  }
  st->passes += 1;
  st->evals += a.n * (long long)K;
  st->last_td = td;
  if (st->mode == kModeFinalAssign || st->mode == kModeAssignOnly) {
    st->total = td;
    st->act = 0;
    st->done = 1;
    return;
  }
  if (st->mode == kModeLloydStep) {
    st->total = td;
    st->last_empty = empties;
    set_action(st, kActUpdate);
    st->done = 1;
    return;
  }
  // ---- convergence test (core.py:342-356)
  const double p = st->td_prev;
  bool conv;
  if (isinf(p))
    conv = false;
  else if (p == 0.0)
    conv = true;
  else
    conv = __ddiv_rn(__dsub_rn(p, td), p) <= st->eps;
  if (conv) {
    // history rows of a converged pass carry empty_cells = 0 (core.py:395-397)
    record_hist(st, K, st->iteration, td, 0);
    if (K < st->target) {
      set_action(st, kActSplit);
    } else {
      st->act = 0;
      st->total = td;
      st->done = 1;
    }
    return;
  }
  record_hist(st, K, st->iteration, td, empties);
  st->td_prev = td;
  st->iteration += 1;
  if (st->iteration > st->max_iter) {
    // guard exhausted: a warning, and the level ends with the UPDATED
    // codebook while the total stays the pre-update TD (core.py:400-417)
    if (st->n_warn < kMaxWarn) st->warn_sizes[st->n_warn] = K;
    st->n_warn += 1;
    if (K < st->target) {
      set_action(st, kActUpdate | kActSplit);
    } else {
      set_action(st, kActUpdate);
      st->total = td;
      st->done = 1;
    }
  } else {
    set_action(st, kActUpdate);
  }
}

__global__ void __launch_bounds__(256) finalize_kernel(KernelArgs a, int phase) {
  pdl_wait();
  if (pass_off(a.st)) return;
  finalize_body(a, phase);
}

// ---------------------------------------------------------------------------
// apply: one thread per source codevector.  Update (update_rows,
// _kernels.py:59-66: sum / n with the int64 fixed-point sum, empty cells keep
// the old row), split (core.py:277-281: rows 2i = c + delta, 2i+1 = c - delta)
// or both, into the other codebook buffer, plus the centred FP32 staging of
// the new rows for the next candidate pass.  Idempotent (speculative passes
// after `done` may repeat it harmlessly).
// ---------------------------------------------------------------------------

// Warp-cooperative staging of destination row k (lane l holds dimension l,
// l + 32, ...): FP32 w = -2 c~ and ||c~||^2 for the FP32 pass, the fp16 hi/lo
// operand image for the TC pass (stage_tc_row's layout).
__device__ __forceinline__ void stage_row_warp(const KernelArgs& a, long long k, const double* row, int dim,
                                               int lane) {
  // row has `dim` values; the staging is zero-padded to the candidate width
  const int cdim = a.cdim;
  double part = 0.0;
  float wv[2] = {0.f, 0.f};
  for (int l = lane, t = 0; l < cdim; l += 32, ++t) {
    const float c = l < dim ? (float)(row[l] - (double)a.mu[l]) : 0.0f;
    part += (double)c * (double)c;
    const float w = -2.0f * c;
    a.w[k * cdim + l] = w;
    if (t < 2) wv[t] = w;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  if (lane == 0) a.nrm[k] = (float)part;
  if (!a.tcb || cdim > 64 || (cdim % 16) != 0) return;
  DevState* st = a.st;
  unsigned short* img = a.tcb + (k / kTcChunk) * tc_chunk_elems(cdim);
  const int r = (int)(k % kTcChunk);
  unsigned short* wh = img;
  unsigned short* wl = img + (long long)kTcChunk * cdim;
  unsigned short* wn = img + 2LL * kTcChunk * cdim;
  const float sw = ldexpf(1.0f, st->tc_ew);
  bool bad = false;
  for (int l = lane, t = 0; l < cdim; l += 32, ++t) {
    const float v = wv[t] * sw;
    const __half h = __float2half_rn(v);
    const __half lo = __float2half_rn(v - __half2float(h));
    bad |= !(fabsf(v) <= 60000.0f);
    wh[tc_off(r, l, cdim)] = __half_as_ushort(h);
    wl[tc_off(r, l, cdim)] = __half_as_ushort(lo);
  }
  if (lane < 16) {
    unsigned short val = 0;
    if (lane < 2) {
      const double nv = ldexp(part, st->tc_ey + st->tc_ew - st->tc_kn);
      const __half nh = __double2half(nv);
      bad |= lane == 0 && !(fabs(nv) <= 60000.0);
      val = lane == 0 ? __half_as_ushort(nh) : __half_as_ushort(__double2half(nv - (double)__half2float(nh)));
    }
    wn[tc_off(r, lane, 16)] = val;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) st->tc_bad = 1;
}

// apply: one warp per source codevector, lanes over dimensions.  Update
// (update_rows, _kernels.py:59-66: sum / n with the int64 fixed-point sum,
// empty cells keep the old row), split (core.py:277-281: rows 2i = c + delta,
// 2i+1 = c - delta) or both, into the other codebook buffer, then the staging
// of the new rows for the next candidate pass.  Idempotent (speculative
// passes after `done` may repeat it harmlessly).
// The codebook work of a pass over any grid: one warp per source codevector.
// zero_lo: consume (read, then clear) the pass's low words -- the fused pass,
// whose action runs exactly once, uses it; the kernel form is idempotent.
__device__ void apply_body(const KernelArgs& a, int stage, bool zero_lo) {
  const DevState* st = a.st;
  const int act = st->act;
  // zero the distortion tiles (other ranks' slots must be 0 before the next
  // allreduce); finalize has consumed them
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.ex.ntiles;
       i += (long long)gridDim.x * blockDim.x)
    a.ex.td()[i] = 0;
  if (act == 0) return;
  const int K = st->act_k;
  const int dim = a.dim;
  const double* src = a.cb[st->act_src];
  double* dst = a.cb[st->act_src ^ 1];
  const int t_lo = st->lo_shift;
  const double delta = st->delta;
  const int ordered = st->ordered;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long k = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); k < K; k += warps) {
    const long long cnt = (act & kActUpdate) ? a.ex.counts()[k] : 0;
    for (int l = lane; l < dim; l += 32) {
      const long long i = k * dim + l;
      double v = src[i];
      const long long lo = a.ex.lo()[i];
      if (zero_lo && lo) a.ex.lo()[i] = 0;  // consumed: the next pass adds from zero
      if ((act & kActUpdate) && cnt > 0)
        v = ordered ? a.ord[i]
                    : __ddiv_rn(fixed_to_double(a.ex.sums()[i], lo, t_lo, -(a.cshift[l] + t_lo)), (double)cnt);
      if (act & kActSplit) {
        dst[(2 * k) * dim + l] = __dadd_rn(v, delta);
        dst[(2 * k + 1) * dim + l] = __dsub_rn(v, delta);
      } else {
        dst[k * dim + l] = v;
      }
    }
    if (stage) {
      __syncwarp();
      if (act & kActSplit) {
        stage_row_warp(a, 2 * k, dst + (2 * k) * dim, dim, lane);
        stage_row_warp(a, 2 * k + 1, dst + (2 * k + 1) * dim, dim, lane);
      } else {
        stage_row_warp(a, k, dst + k * dim, dim, lane);
      }
    }
  }
}

__global__ void __launch_bounds__(256) apply_kernel(KernelArgs a, int stage) {
  pdl_wait();
  if (a.st->skip) return;  // (not `done`: speculative passes re-apply harmlessly)
  apply_body(a, stage, false);
}

// ---------------------------------------------------------------------------
// Fused pass for small codebooks (K <= 512 / L): ONE cooperative persistent
// kernel does the whole training pass -- FP32 candidate pass + certification,
// the reference's FP64 scan for the rows it cannot certify (a warp per row,
// lanes = codevectors), exact winner distances, the distortion tile partials
// in the fixed tree of td_tiles_kernel, two-word cell sums in half-warp
// tables, the slab reduction, finalize (one block) and apply (all blocks) --
// separated by three grid barriers.  Each row is read from HBM once.  The
// per-kernel path of the same pass sees `skip` and idles (one graph serves
// every level).  Reference: _kernels.py:18-66, core.py:384-415.
// ---------------------------------------------------------------------------
constexpr int kFuseThreads = 512;
template <int L>
__host__ __device__ constexpr int fused_kmax() { return 512 / L; }

// grid-wide barrier (cooperative launch: every CTA is resident)
__device__ __forceinline__ void grid_sync(DevState* st) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* genp = &st->bar_gen;
    const unsigned g = *genp;
    __threadfence();
    if (atomicAdd(&st->bar_count, 1u) == gridDim.x - 1) {
      st->bar_count = 0;
      __threadfence();
      atomicAdd(&st->bar_gen, 1u);
    } else {
      while (*genp == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int L>
struct FuseSmem {
  static constexpr int KF = fused_kmax<L>();
  float w[KF * L];
  float nrm[KF];
  double cb[KF * L];
  long long tab[32][KF * L];   // half-warp tables (2 per warp)
  unsigned tcnt[32][KF];
  double red[32];
};

// reference-arithmetic distance of a row (x32 / x64, dim values) to a
// codevector staged in shared memory, 16 values loaded at a time
template <typename XT>
__device__ __forceinline__ double smem_dist(const XT* __restrict__ x, const double* c, int dim) {
  double d = 0.0;
  for (int c0 = 0; c0 < dim; c0 += 16) {
    XT xr[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) xr[l] = c0 + l < dim ? x[c0 + l] : (XT)0;
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      if (c0 + l < dim) {
        const double diff = __dsub_rn((double)xr[l], c[c0 + l]);
        d = __dadd_rn(d, __dmul_rn(diff, diff));
      }
    }
  }
  return d;
}

// Phase A of the fused pass, warp-independent: the grid's warps take
// 128-row chunks round-robin (lane: rows base + lane + 32 k, k < 4): the
// candidate pass and certification (assign_chunk's arithmetic and band),
// the reference's FP64 scan for rows the band cannot certify (lanes =
// codevectors, lexicographic (d, j) minimum), exact winner distances,
// cells / distances out, and the two-word cell sums into the warp's
// half-warp tables (lanes = dimensions, 16 rows' values loaded together, runs
// of one cell summed in registers).  No block-wide synchronisation.
template <int L, typename XT>
__device__ __forceinline__ void fused_rows(const KernelArgs& a, const XT* __restrict__ X, FuseSmem<L>& sm,
                                           int K, int t_lo, int metric, const float (&mu)[L]) {
  constexpr int kChunk = 128, R = 4;
  constexpr int RB = L == 16 ? 4 : (L == 32 ? 2 : 1);
  const int dim = a.dim;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, hl = lane & 15;
  long long* tab = sm.tab[2 * warp + half];
  unsigned* tcnt = sm.tcnt[2 * warp + half];
  const float u = 5.9604645e-8f;
  const long long nchunks = (a.n + kChunk - 1) / kChunk;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  int nflag = 0;
  for (long long ch = gw; ch < nchunks; ch += nw) {
    const long long base = ch * kChunk;
    int cell[R];
    double dist[R];
    unsigned flagm = 0;  // bit k: row k of this lane needs the exact scan
#pragma unroll 1
    for (int kb = 0; kb < R; kb += RB) {
      float y[RB][L];
      float q[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const long long row = base + lane + 32 * (kb + k);
        const float4* src = reinterpret_cast<const float4*>(a.xc + (row < a.n ? row : base) * L);
#pragma unroll
        for (int v = 0; v < L / 4; ++v) {
          const float4 t4 = __ldg(src + v);
          y[k][4 * v + 0] = t4.x;
          y[k][4 * v + 1] = t4.y;
          y[k][4 * v + 2] = t4.z;
          y[k][4 * v + 3] = t4.w;
        }
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        q[k] = 0.f;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          y[k][l] = __fsub_rn(y[k][l], mu[l]);
          q[k] = fmaf(y[k][l], y[k][l], q[k]);
        }
      }
      float m1[RB], m2[RB];
      int i1[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        m1[k] = INFINITY;
        m2[k] = INFINITY;
        i1[k] = 0;
      }
#pragma unroll 1
      for (int j = 0; j < K; ++j) {
        float v[RB];
        const float nj = sm.nrm[j];
#pragma unroll
        for (int k = 0; k < RB; ++k) v[k] = nj;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          const float wl = sm.w[j * L + l];
#pragma unroll
          for (int k = 0; k < RB; ++k) v[k] = fmaf(wl, y[k][l], v[k]);
        }
#pragma unroll
        for (int k = 0; k < RB; ++k) {
          const float n2 = fminf(m2[k], fmaxf(m1[k], v[k]));
          const bool p = v[k] < m1[k];
          m1[k] = fminf(m1[k], v[k]);
          i1[k] = p ? j : i1[k];
          m2[k] = n2;
        }
      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const long long row = base + lane + 32 * (kb + k);
        const float yn = sqrtf(q[k]);
        const float d2 = fmaxf(m2[k] + q[k], 0.f);
        const float sd = sqrtf(d2) * 1.01f + 1.0f;
        const float Sm = 2.02f * yn + sd;
        const float E = (float)(L + 3) * u * Sm * Sm + 2.5f * u * sd * Sm + 1e-14f * Sm * Sm;
        const float band = 3.0f * E + input_band(row < a.n ? rin_of(a, row) : 0.f, m1[k] + q[k], 3.0f * E);
        const bool ok = row >= a.n || (m2[k] - m1[k]) > band;
#pragma unroll
        for (int kk = 0; kk < R; ++kk)
          if (kk == kb + k) cell[kk] = i1[k];
        if (!ok) flagm |= 1u << (kb + k);
      }
    }
    // exact distances of the certified winners (the rows the reference sees)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const long long row = base + lane + 32 * k;
      dist[k] = (row < a.n && !(flagm >> k & 1)) ? smem_dist(X + row * dim, sm.cb + cell[k] * dim, dim) : 0.0;
    }
    // rows the band could not certify: the warp scans each in FP64
#pragma unroll
    for (int k = 0; k < R; ++k) {
      unsigned fl = __ballot_sync(0xffffffffu, (flagm >> k) & 1);
      nflag += __popc(fl);
      while (fl) {
        const int src = __ffs(fl) - 1;
        fl &= fl - 1;
        const long long row = base + src + 32 * k;
        double d = INFINITY;
        int j = lane;
        if (lane < K) {
          d = smem_dist(X + row * dim, sm.cb + lane * dim, dim);
          if (!(d < INFINITY)) d = INFINITY;  // NaN / inf never win a strict <
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double od = __shfl_xor_sync(0xffffffffu, d, off);
          const int oj = __shfl_xor_sync(0xffffffffu, j, off);
          if (od < d || (od == d && oj < j)) {
            d = od;
            j = oj;
          }
        }
        if (lane == src) {
          cell[k] = d < INFINITY ? j : 0;
          dist[k] = d;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const long long row = base + lane + 32 * k;
      if (row >= a.n) continue;
      a.idx[row] = cell[k];
      if (a.dists) a.dists[row] = metric == kEuclidean ? sqrt(dist[k]) : dist[k];
    }
    // two-word cell sums: 32 rows (k) at a time, half-warp h takes row 2p + h
#pragma unroll 1
    for (int k = 0; k < R; ++k) {
      for (int c0 = 0; c0 < dim; c0 += 16) {
        const int l = c0 + hl;
        const bool lon = l < dim;
        const int shl = lon ? __ldg(a.cshift + l) : 0;
        XT xv[16];
        int cv[16];
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          const int rl = 2 * p + half;  // row base + rl + 32 k, held by lane rl
          const long long row = base + rl + 32 * k;
          int c = 0;
#pragma unroll
          for (int kk = 0; kk < R; ++kk) c = kk == k ? __shfl_sync(0xffffffffu, cell[kk], rl) : c;
          const bool ok = row < a.n;
          cv[p] = ok ? c : -1;
          xv[p] = (ok && lon) ? X[row * dim + l] : (XT)0;
        }
        long long acc = 0, acc_lo = 0;
        int cur = -1;
        unsigned run = 0;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          if (cv[p] != cur) {  // uniform within the half-warp (one row)
            if (cur >= 0) {
              if (lon) {
                tab[cur * L + l] += acc;
                add_lo(a, cur, l, acc_lo);
              }
              if (c0 == 0 && hl == 0) tcnt[cur] += run;
            }
            cur = cv[p];
            acc = 0;
            acc_lo = 0;
            run = 0;
          }
          if (cur >= 0) {
            long long h, lo2;
            split_fixed(xv[p], shl, t_lo, h, lo2);
            acc += h;
            acc_lo += lo2;
            ++run;
          }
        }
        if (cur >= 0) {
          if (lon) {
            tab[cur * L + l] += acc;
            add_lo(a, cur, l, acc_lo);
          }
          if (c0 == 0 && hl == 0) tcnt[cur] += run;
        }
      }
    }
  }
  if (lane == 0 && nflag) atomicAdd(&a.st->flag_count, nflag);
}

template <int L, typename XT>
__device__ __forceinline__ void fused_pass(const KernelArgs& a, const XT* __restrict__ X) {
  using S = FuseSmem<L>;
  constexpr int KF = S::KF;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);
  DevState* st = a.st;
  const int K = st->size;
  const int dim = a.dim;
  const int tid = threadIdx.x;
  const double* cbg = a.cb[st->cur];
  for (int i = tid; i < K * L; i += blockDim.x) sm.w[i] = a.w[i];
  for (int i = tid; i < K; i += blockDim.x) sm.nrm[i] = a.nrm[i];
  for (int i = tid; i < K * dim; i += blockDim.x) sm.cb[i] = cbg[i];
  for (int i = tid; i < 32 * KF * L; i += blockDim.x) (&sm.tab[0][0])[i] = 0;
  for (int i = tid; i < 32 * KF; i += blockDim.x) (&sm.tcnt[0][0])[i] = 0;
  float mu[L];
#pragma unroll
  for (int l = 0; l < L; ++l) mu[l] = a.mu[l];
  __syncthreads();
  fused_rows<L, XT>(a, X, sm, K, st->lo_shift, st->metric, mu);
  __syncthreads();
  // this CTA's slab: its half-warp tables summed (int64, any order exact)
  long long* slab = a.partials + (long long)blockIdx.x * ((long long)a.kmax * dim + a.kmax);
  for (int i = tid; i < K * dim; i += blockDim.x) {
    const int c = i / dim, l = i % dim;
    long long v = 0;
    for (int tb2 = 0; tb2 < 32; ++tb2) v += sm.tab[tb2][c * L + l];
    slab[i] = v;
  }
  for (int c = tid; c < K; c += blockDim.x) {
    long long v = 0;
    for (int tb2 = 0; tb2 < 32; ++tb2) v += sm.tcnt[tb2][c];
    slab[(long long)K * dim + c] = v;
  }
}

// the distortion partial of 2048-row tile t from the stored distances, in
// td_tiles_kernel's order (threads 0..255 of the block)
__device__ __forceinline__ void tile_partial(const KernelArgs& a, long long t, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 256) {
    double sacc = 0.0;
#pragma unroll
    for (int r = 0; r < kTdTile / 256; ++r) {
      const long long row = t * kTdTile + (long long)r * 256 + tid;
      sacc = __dadd_rn(sacc, row < a.n ? a.dists[row] : 0.0);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sacc = __dadd_rn(sacc, __shfl_xor_sync(0xffffffffu, sacc, off));
    if (lane == 0) red[warp] = sacc;
  }
  __syncthreads();
  if (tid == 0) {
    double t2 = 0.0;
    for (int w = 0; w < 8; ++w) t2 = __dadd_rn(t2, red[w]);
    a.ex.td()[a.tile0 + t] = __double_as_longlong(t2);
  }
  __syncthreads();
}

template <int L>
__global__ void __launch_bounds__(kFuseThreads, 1) pass_small_kernel(KernelArgs a) {
  DevState* st = a.st;
  if (st->done) return;
  const int K = st->size;
  if (st->mode != kModeTrain || st->ordered || K > fused_kmax<L>()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->skip = 0;  // the per-kernel path runs this pass
    return;
  }
  if (a.x64)
    fused_pass<L, double>(a, a.x64);
  else
    fused_pass<L, float>(a, a.x32);
  grid_sync(st);
  // distortion tile partials (every row's distance is stored now)
  {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* red = reinterpret_cast<FuseSmem<L>*>(smem_raw)->red;
    const long long ntiles = (a.n + kTdTile - 1) / kTdTile;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) tile_partial(a, t, red);
  }
  // slabs -> the exchange buffer (fixed order over CTAs; integer sums)
  {
    const int dim = a.dim;
    const long long words = (long long)K * dim + K;
    const long long stride = (long long)a.kmax * dim + a.kmax;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < words;
         w += (long long)gridDim.x * blockDim.x) {
      long long v = 0;
      for (int b = 0; b < (int)gridDim.x; ++b) v += a.partials[(long long)b * stride + w];
      if (w < (long long)K * dim)
        a.ex.sums()[w] = v;
      else
        a.ex.counts()[w - (long long)K * dim] = v;
    }
  }
  grid_sync(st);
  if (blockIdx.x == 0) {
    finalize_body(a, 1, false);
    if (threadIdx.x == 0) st->skip = 1;  // the rest of this pass's kernels idle
  }
  grid_sync(st);
  apply_body(a, 1, true);
}

// Launch the fused pass (one CTA per SM, cooperative); it returns at once
// for passes it does not take.  Opt-in (VQB_FUSE=1): measured on the B200 it
// is correct but slower than the per-kernel pass (cfg2 K=2: 177 vs 110 us per
// pass; instruction-bound at 16 warps per SM -- DESIGN.md section 9).
cudaError_t launch_pass_small(const KernelArgs& a, int sms, cudaStream_t s) {
  static const bool on = getenv_flag("VQB_FUSE", 0) != 0;
  if (!on || !a.xc) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(kFuseThreads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.stream = s;
  cudaError_t e = cudaSuccess;
  switch (a.cdim) {
#define VQB_FUSE_L(LL)                                                                                      \
  case LL: {                                                                                                \
    cfg.dynamicSmemBytes = sizeof(FuseSmem<LL>);                                                            \
    e = cudaFuncSetAttribute(pass_small_kernel<LL>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                             (int)sizeof(FuseSmem<LL>));                                                    \
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, pass_small_kernel<LL>, a);                           \
    break;                                                                                                  \
  }
    VQB_FUSE_L(16)
    VQB_FUSE_L(32)
    VQB_FUSE_L(64)
#undef VQB_FUSE_L
    default: return cudaSuccess;
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_finalize(const KernelArgs& a, bool stage, cudaStream_t s) {
  {
    cudaError_t e1 = launch_k(finalize_kernel, 1, 256, 0, s, a, 1);
    if (e1 != cudaSuccess) return e1;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int blocks = (int)((a.kmax + 7) / 8);  // one warp per codevector
  if (blocks < 8) blocks = 8;
  {
    cudaError_t e1 = launch_k(apply_kernel, blocks, 256, 0, s, a, stage ? 1 : 0);
    if (e1 != cudaSuccess) return e1;
  }
  return cudaGetLastError();
}

cudaError_t launch_init_centroid(const KernelArgs& a, bool stage, cudaStream_t s) {
  {
    cudaError_t e1 = launch_k(finalize_kernel, 1, 256, 0, s, a, 0);
    if (e1 != cudaSuccess) return e1;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  {
    cudaError_t e1 = launch_k(apply_kernel, 8, 256, 0, s, a, stage ? 1 : 0);
    if (e1 != cudaSuccess) return e1;
  }
  // the column sums' low words are consumed: clear them (the fused pass adds
  // from zero and clears after itself)
  e = launch_k(zero_lo_kernel, 64, 256, 0, s, a, 0);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// staging padding (rows >= K never win) and a clean exchange buffer
__global__ void clear_kernel(KernelArgs a) {
  pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.ex.words();
       i += (long long)gridDim.x * blockDim.x)
    a.ex.base[i] = 0;
  const long long kpad = (a.kmax + 3) / 4 * 4;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < kpad;
       k += (long long)gridDim.x * blockDim.x) {
    a.nrm[k] = INFINITY;
    for (int l = 0; l < a.cdim; ++l) a.w[k * a.cdim + l] = 0.0f;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.st->flag_count = 0;
    a.st->flag2_count = 0;
  }
}

cudaError_t launch_clear(const KernelArgs& a, cudaStream_t s) {
  {
    cudaError_t e1 = launch_k(clear_kernel, 64, 256, 0, s, a);
    if (e1 != cudaSuccess) return e1;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------

template <typename T>
__global__ void maxabs_kernel(const T* x, long long count, unsigned long long* out) {
  double m = 0.0;
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    double v = fabs((double)x[i]);
    if (!(v <= DBL_MAX)) bad = true;
    m = fmax(m, v);
  }
  unsigned long long bits = bad ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(m);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    unsigned long long o = __shfl_xor_sync(0xffffffffu, bits, off);
    bits = o > bits ? o : bits;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, bits);
}

cudaError_t launch_maxabs(const float* x32, const double* x64, long long count,
                          unsigned long long* out_bits, int sms, cudaStream_t s) {
  if (x32)
    maxabs_kernel<float><<<sms * 4, 256, 0, s>>>(x32, count, out_bits);
  else
    maxabs_kernel<double><<<sms * 4, 256, 0, s>>>(x64, count, out_bits);
  return cudaGetLastError();
}

// Per-column statistics of a row block for the two-word fixed-point plan:
// max |x| (FP64 bit patterns; NaN bits when a value is not finite) and the
// exponent of the lowest set bit (INT_MAX when the column is all zeros).
// Thread t keeps column t % dim when the grid's thread count is a multiple of
// dim (dim divides 256), else it walks elements with shared-memory atomics.
__device__ __forceinline__ int lowbit_exp(float x) {
  const unsigned u = __float_as_uint(x);
  const unsigned E = (u >> 23) & 0xffu;
  unsigned m = u & 0x7fffffu;
  if (E == 0xffu) return INT_MIN;  // non-finite: flagged through the max
  int e0 = -149;
  if (E) {
    m |= 0x800000u;
    e0 = (int)E - 150;
  }
  return m ? e0 + __ffs((int)m) - 1 : INT_MAX;
}
__device__ __forceinline__ int lowbit_exp(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  const unsigned E = (unsigned)((u >> 52) & 0x7ffu);
  unsigned long long m = u & 0xfffffffffffffull;
  if (E == 0x7ffu) return INT_MIN;
  int e0 = -1074;
  if (E) {
    m |= 1ull << 52;
    e0 = (int)E - 1075;
  }
  return m ? e0 + __ffsll((long long)m) - 1 : INT_MAX;
}

template <typename T>
__global__ void __launch_bounds__(256) colstats_kernel(const T* __restrict__ x, long long rows, int dim,
                                                       unsigned long long* cmax, int* clow) {
  const long long count = rows * dim;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (stride % dim == 0) {
    double m = 0.0;
    bool bad = false;
    int low = INT_MAX;
    for (long long i = i0; i < count; i += stride) {
      const T v = x[i];
      const double av = fabs((double)v);
      bad |= !(av <= DBL_MAX);
      m = fmax(m, av);
      low = min(low, lowbit_exp(v));
    }
    if (i0 < count) {
      const int c = (int)(i0 % dim);
      atomicMax(cmax + c, bad ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(m));
      if (low != INT_MAX) atomicMin(clow + c, low);
    }
    return;
  }
  for (long long i = i0; i < count; i += stride) {
    const T v = x[i];
    const double av = fabs((double)v);
    const int c = (int)(i % dim);
    atomicMax(cmax + c, !(av <= DBL_MAX) ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(av));
    const int low = lowbit_exp(v);
    if (low != INT_MAX) atomicMin(clow + c, low);
  }
}

__global__ void colstats_reset_kernel(unsigned long long* cmax, int* clow, int dim) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < dim; c += gridDim.x * blockDim.x) {
    cmax[c] = 0;
    clow[c] = INT_MAX;
  }
}

cudaError_t launch_colstats_reset(unsigned long long* cmax, int* clow, int dim, cudaStream_t s) {
  colstats_reset_kernel<<<(dim + 255) / 256, 256, 0, s>>>(cmax, clow, dim);
  return cudaGetLastError();
}

cudaError_t launch_colstats(const float* x32, const double* x64, long long rows, int dim,
                            unsigned long long* cmax, int* clow, int sms, cudaStream_t s) {
  if (rows < 1) return cudaSuccess;
  const long long count = rows * dim;
  long long blocks = (count + 255) / 256;
  const long long cap = (long long)sms * 8;
  if (blocks > cap) blocks = cap;
  if (x32)
    colstats_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(x32, rows, dim, cmax, clow);
  else
    colstats_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(x64, rows, dim, cmax, clow);
  return cudaGetLastError();
}

// fixed-point plan from column stats, on the device (the host-buffer Lloyd
// step needs no host round trip): cshift, lo_shift, exactness flags, and the
// overall max |x| for the non-finite check
__global__ void set_shift_kernel(DevState* st, const unsigned long long* cmax, const int* clow, int dim,
                                 long long n_global, int* cshift, unsigned long long* maxabs_bits) {
  __shared__ int s_exact, s_ref, s_bad;
  if (threadIdx.x == 0) {
    s_exact = 1;
    s_ref = 1;
    s_bad = 0;
  }
  __syncthreads();
  unsigned long long mb = 0;
  for (int c = threadIdx.x; c < dim; c += blockDim.x) {
    const double m = __longlong_as_double((long long)cmax[c]);
    const FixedCol f = fixed_plan(n_global, m, clow[c]);
    cshift[c] = f.s;
    if (!f.exact) atomicAnd(&s_exact, 0);
    if (!f.ref_exact) atomicAnd(&s_ref, 0);
    if (!(m <= DBL_MAX)) atomicOr(&s_bad, 1);
    mb = cmax[c] > mb ? cmax[c] : mb;
  }
  if (maxabs_bits) atomicMax(maxabs_bits, mb);
  __syncthreads();
  if (threadIdx.x == 0) {
    st->lo_shift = fixed_lo_shift(n_global);
    st->sums_exact = s_exact;
    st->ref_exact = s_ref;
    st->nonfinite = s_bad;
  }
}

cudaError_t launch_set_shift(DevState* st, const unsigned long long* cmax, const int* clow, int dim,
                             long long n_global, int* cshift, unsigned long long* maxabs_bits, cudaStream_t s) {
  set_shift_kernel<<<1, 256, 0, s>>>(st, cmax, clow, dim, n_global, cshift, maxabs_bits);
  return cudaGetLastError();
}

__global__ void widen_idx_kernel(const int* idx, long long* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = idx[i];
}

cudaError_t launch_widen_idx(const int* idx, long long* out, long long n, int sms, cudaStream_t s) {
  widen_idx_kernel<<<sms * 4, 256, 0, s>>>(idx, out, n);
  return cudaGetLastError();
}

__global__ void sum_inorder_kernel(const double* v, long long n, double* out) {
  double s = 0.0;
  for (long long i = 0; i < n; ++i) s = __dadd_rn(s, v[i]);
  *out = s;
}

cudaError_t launch_sum_inorder(const double* v, long long n, double* out, cudaStream_t s) {
  sum_inorder_kernel<<<1, 1, 0, s>>>(v, n, out);
  return cudaGetLastError();
}

// reset the per-call state (one-shot assign / update / Lloyd step calls)
__global__ void reset_kernel(DevState* st, int mode, int size, int metric, int ordered,
                             int keep_cur) {
  pdl_wait();
  st->mode = mode;
  st->size = size;
  st->metric = metric;
  st->ordered = ordered;
  st->done = 0;
  st->skip = 0;
  if (!keep_cur) st->cur = 0;
  st->flag_count = 0;
  st->flag2_count = 0;
  st->iteration = 1;
  st->td_prev = INFINITY;
  if (!keep_cur) {
    st->n_hist = 0;
    st->n_warn = 0;
    st->passes = 0;
    st->evals = 0;
    st->flagged_total = 0;
    st->flagged2_total = 0;
  }
}

cudaError_t launch_reset(DevState* st, int mode, int size, int metric, int ordered, int keep_cur,
                         cudaStream_t s) {
  {
    cudaError_t e1 = launch_k(reset_kernel, 1, 1, 0, s, st, mode, size, metric, ordered, keep_cur);
    if (e1 != cudaSuccess) return e1;
  }
  return cudaGetLastError();
}

__global__ void cells_to_idx_kernel(const long long* cells, int* idx, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    idx[i] = (int)cells[i];
}

cudaError_t launch_cells_to_idx(const long long* cells, int* idx, long long n, int sms, cudaStream_t s) {
  cells_to_idx_kernel<<<sms * 4, 256, 0, s>>>(cells, idx, n);
  return cudaGetLastError();
}

// float64 rows that are exactly float32 (the usual case: TrainingSet widens
// float32 / 8-bit data, core.py:47-60) take the FP32 candidate path.
__global__ void f64_to_f32_kernel(const double* x64, float* x32, long long count, int* inexact) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = x64[i];
    const float f = (float)v;
    x32[i] = f;
    if (!((double)f == v)) bad = 1;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(inexact, 1);
}

cudaError_t launch_f64_to_f32_exact(const double* x64, float* x32, long long count, int* inexact,
                                    int sms, cudaStream_t s) {
  f64_to_f32_kernel<<<sms * 4, 256, 0, s>>>(x64, x32, count, inexact);
  return cudaGetLastError();
}

// _kernels.column_sums (_kernels.py:81-89): ascending rows, one thread per column
template <typename XT>
__global__ void column_sums_kernel(const XT* x, long long m, int dim, double* out) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= dim) return;
  double s = 0.0;
  for (long long j = 0; j < m; ++j) s = __dadd_rn(s, load_x(x, j * dim + l));
  out[l] = s;
}

cudaError_t launch_column_sums_ordered(const double* x64, const float* x32, long long m, int dim,
                                       double* out, cudaStream_t s) {
  const int blocks = (dim + 63) / 64;
  if (x32)
    column_sums_kernel<float><<<blocks, 64, 0, s>>>(x32, m, dim, out);
  else
    column_sums_kernel<double><<<blocks, 64, 0, s>>>(x64, m, dim, out);
  return cudaGetLastError();
}

// Candidate rows: fl32 of each value, zero-padded to cdim; for float64 rows
// also rin = 2^-24 ||x|| (x 1.0001, + a subnormal floor), the bound of the
// rounding ||x - fl32(x)|| the certified band widens by (input_band)
template <typename XT>
__global__ void candidate_rows_kernel(const XT* __restrict__ x, long long n, int dim, int cdim, float* xc,
                                      float* rin) {
  for (long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x; row < n;
       row += (long long)gridDim.x * blockDim.x) {
    double nn = 0.0;
    for (int l = 0; l < cdim; ++l) {
      const double v = l < dim ? (double)x[row * dim + l] : 0.0;
      xc[row * cdim + l] = (float)v;
      nn += v * v;
    }
    if (rin) rin[row] = (float)(sqrt(nn) * 5.9604644775390625e-8 * 1.0001 + 1e-37);
  }
}

cudaError_t launch_candidate_rows(const float* x32, const double* x64, long long n, int dim, int cdim,
                                  float* xc, float* rin, int sms, cudaStream_t s) {
  if (x64)
    candidate_rows_kernel<double><<<sms * 8, 256, 0, s>>>(x64, n, dim, cdim, xc, rin);
  else
    candidate_rows_kernel<float><<<sms * 8, 256, 0, s>>>(x32, n, dim, cdim, xc, nullptr);
  return cudaGetLastError();
}

// _kernels.pair_distance (_kernels.py:69-78)
__global__ void pair_distance_kernel(const double* a, const double* b, int dim, int metric,
                                     double* out) {
  double d = ref_dist(a, b, dim);
  *out = metric == kEuclidean ? sqrt(d) : d;
}

cudaError_t launch_pair_distance(const double* a, const double* b, int dim, int metric, double* out,
                                 cudaStream_t s) {
  pair_distance_kernel<<<1, 1, 0, s>>>(a, b, dim, metric, out);
  return cudaGetLastError();
}

}  // namespace vqb
