// Tensor-core candidate pass for the nearest-codevector search (sm_100a,
// tcgen05 + TMEM).  Reference: _kernels.assign_range (_kernels.py:18-36).
//
// The distance pass is GEMM-shaped: for a tile of 128 rows and a chunk of
// 256 codewords, v_ij = ||c~_j||^2 - 2 y~_i . c~_j is one M=128 x N=256 MMA
// with K = L.  FP32-level accuracy comes from an fp16 hi/lo split of both
// operands (y = yh + yl, w = wh + wl; the yl.wl term is below 2^-44) and the
// norm folded in as an extra K-step (a constant column 2^kn times nh + nl):
//
//   D = yh.wh + yh.wl + yl.wh + 2^kn (nh + nl) = 2^(ey+ew) v      (fp32, TMEM)
//
// so the epilogue only does the minimum / band bookkeeping on values read
// straight from TMEM (per value half a 3-input FMNMX for the chunk minimum,
// then one FSETP + predicated add for the count inside the band).  The
// certification band is the FP32 one widened for the split (4 x 2^-22) and
// for tensor-core accumulation (2 x 2^-22 of the magnitude sum per MMA
// instruction; tools/tc_probe.py measures <= 0.5 x 2^-22 per MMA against a
// float64 emulation of the same operands); rows that do not certify go to the
// same shortlist / FP64 re-rank as the FP32 pass, so a certified index is the
// reference's index.
//
// CTA (persistent, one per SM, over 128-row tiles) = 1 MMA-issuer warp +
// 16 (L = 16) or 8 epilogue warps (4 lane quarters x column parts) + a
// streamer / converter pair + 8 certification warps (two groups of 4).  The
// codebook's operand image (staged by apply_kernel / prep_codebook in the
// exact smem layout) is bulk-copied into smem once, or streamed through a TMA
// ring when it does not fit; row tiles come from the prebuilt fp16 row image
// of a resident training set (bulk copies) or are converted from x32;
// accumulators are double-buffered in TMEM (2 x 256 columns), so the MMAs of
// chunk c+1 overlap the epilogue of chunk c.  The certification warps merge
// the parts' results, compute the certified row's exact FP64 distance and
// queue the rest, off the epilogue's critical path.
#include <cfloat>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>

#include "ptx.h"
#include "refarith.cuh"
#include "vqb200_internal.h"

namespace vqb {

// suspend-time hint of the certification warps' wait for tile results
#ifndef VQB_SLEEP_NS
#define VQB_SLEEP_NS 20000
#endif
constexpr uint32_t kSleepNs = VQB_SLEEP_NS;
// epilogue TMEM reads: 32-column loads double-buffered in registers (the next
// group's load in flight while this one is scanned), or waited on at once.
// Pipelining pays with 8 epilogue warps (L >= 32: cfg3 pass -5 %); with 16
// (L = 16) the warps already hide the load latency and 64 value registers do
// not fit.
// VQB_PIPE_LD=0/1 forces one form (A/B builds).
#ifndef VQB_PIPE_LD
#define VQB_PIPE_LD -1
#endif
template <int L>
__host__ __device__ constexpr bool pipe_ld() { return VQB_PIPE_LD < 0 ? L >= 32 : VQB_PIPE_LD != 0; }

// certification groups of 4 warps at L >= 32: the role profile showed the
// certification warps busy 94 % at cfg3 (64-dimension FP64 distances) with
// the epilogue waiting on them; a second group cuts the pass 14 % (96
// registers, no spills)
#ifndef VQB_CERT_GROUPS_WIDE
#define VQB_CERT_GROUPS_WIDE 2
#endif
template <int L>
struct TcCfg {
  // epilogue warps: kParts per TMEM lane quarter, each scanning 256 / kParts
  // columns of every chunk (more warps hide the argmin chains' latency; L=16
  // has the registers for 16)
  static constexpr int kEpiWarps = L == 16 ? 16 : 8;
  static constexpr int kParts = kEpiWarps / 4;
  static constexpr int kSpan = kTcChunk / kParts;
  // Warp roles: 0 issues MMAs; 1..kEpiWarps run the epilogue; kEpiWarps + 1
  // streams codebook chunks when the codebook does not fit in shared memory
  // (else it converts rows); kEpiWarps + 2 and kExtraConv more convert row
  // tiles into the A operand buffers (at small K the conversion is the
  // pipeline's longest stage); then (kTcTop2) kCertGroups x 4 certification
  // warps, one per 32-row quarter, finish each tile's rows (part merge, FP64
  // winner distance, queueing) off the epilogue's critical path.  At L = 64
  // that work (192 FP64 ops + a 768 B gather per row) on epilogue part 0
  // stalled the MMAs 60 % of the time; dedicated warps cut the pass by 13 %.
  static constexpr int kExtraConv = 0;
  static constexpr bool kCertWarps = true;
  static constexpr int kCertGroups = L == 16 ? 2 : VQB_CERT_GROUPS_WIDE;
  // the tile results are double-buffered (res[i & 1]) and each buffer's
  // res_empty barrier expects one group's 4 warps: group g owns buffer g, so
  // a third group would arrive out of phase and deadlock
  static_assert(kCertGroups == 1 || kCertGroups == 2, "certification groups: 1 or 2");
  static constexpr int kCertWarp0 = 3 + kEpiWarps + kExtraConv;
  static constexpr int threads(int mode) {
    return 32 * (kCertWarp0 + (mode == 0 && kCertWarps ? 4 * kCertGroups : 0));
  }
  static constexpr size_t kChunkBytes = (size_t)kTcChunk * (2 * L + 16) * 2;
  static constexpr size_t kABytes = (size_t)kTcRows * (2 * L + 16) * 2;
  static constexpr size_t kMisc = kParts == 4 ? 16384 : 10240;
  // contiguous row tiles arrive by one bulk copy into this stage (L <= 32);
  // the converter then reads shared memory instead of 64 B per lane from HBM
  // (double-buffered at L = 16; sessions with resident rows use the prebuilt
  // row image instead)
  static constexpr int kXsStages = L == 16 ? 2 : 1;
  static_assert(kXsStages <= 4, "xs_full barriers");
  static constexpr size_t kXsTile = (size_t)kTcRows * L * 4;
  static constexpr size_t kXsBytes = L <= 32 ? kXsStages * kXsTile : 0;
  static constexpr size_t kSmemCap = 227 * 1024;
  static constexpr int kMaxChunks = (int)((kSmemCap - 2 * kABytes - kXsBytes - kMisc) / kChunkBytes);
  static constexpr int kStages = kMaxChunks >= 4 ? 4 : kMaxChunks;  // streaming ring
};

int tc_max_size(int dim) {
  // resident codebooks up to kMaxChunks x 256; larger ones stream through the
  // ring (the shortlist merge stores candidates as 16-bit indices)
  switch (dim) {
    case 16: case 32: case 64: return 65536;
    default: return 0;
  }
}

// misc smem: barriers | tmem slot | merge areas
template <int P>
struct TcMisc {
  uint64_t b_full;
  uint64_t bs_full[4];   // streaming ring: chunk landed
  uint64_t bs_empty[4];  // streaming ring: MMAs reading the stage completed
  uint64_t a_full[2];
  uint64_t a_empty[2];
  uint64_t d_full[2];
  uint64_t d_empty[2];
  uint64_t res_full[2];   // epilogue -> certification: tile results in res[i & 1]
  uint64_t res_empty[2];  // certification has read res[i & 1]
  uint32_t tmem;
  uint32_t pad;
  uint64_t q_full[4];      // converter -> epilogue: qrow[i & 3] written
  uint64_t xs_full[4];     // row tile landed in X stage i % kXsStages
  float qrow[4][kTcRows];  // ||y~||^2 per row of tile i (slot i & 3; -1: row out of fp16 range)
  union {
    struct {               // kTcTop2: every part's (minimum, second minimum, index) per row
      float m1[P][kTcRows];
      float m2[P][kTcRows];
      int i1[P][kTcRows];
      float q[kTcRows];
    } res[2];
    struct {                   // kTcShortlist, double-buffered by tile parity
      double best[P][kTcRows];   // every part's best FP64 distance ...
      int bestj[P][kTcRows];     // ... and its index
      unsigned char count[P][kTcRows];  // every part's shortlist size (saturated)
    } sl[2];
  } merge;
};

// Certification band E (unscaled distance units) for a row with minimum
// m1v = ||c||^2 - 2 y.c and q = ||y||^2: fp16 split (4 x 2^-22) and
// tensor-core accumulation (2 x 2^-22 of the magnitude sum per MMA; measured
// <= 0.25 of that, tools/tc_probe.py) of S = 2.02|y| + sd, the FP32 terms,
// and the operands' fp16 quantisation (eyw = sqrt(L) u (2^-ey + 2^-ew)).  sd
// bounds sqrt(distance) of every value inside the band (m1 + 3E, one
// fixed-point step).
template <int L>
__device__ __forceinline__ float tc_band(float m1v, float q, float yn, float eyw) {
  constexpr float u = 5.9604645e-8f;
  // accumulation term per MMA in units of 2^-22 (A/B builds only: the measured
  // worst on band-edge operands is 0.29 of the default 2)
#ifndef VQB_TC_ACC_TERM
#define VQB_TC_ACC_TERM 2
#endif
  constexpr float cacc = (float)(VQB_TC_ACC_TERM * (3 * L / 16 + 1) + 4) * 2.3841858e-7f + 1e-14f;
  const float d1 = fmaxf(m1v + fmaxf(q, 0.f), 0.f);
  auto poly = [&](float sd) {
    const float S = fmaf(2.02f, yn, sd);
    return fmaf(fmaf(cacc, S, 2.5f * u * sd), S, eyw * S);
  };
  const float e0 = poly(fmaf(sqrtf(d1), 1.01f, 1.0f));
  return poly(fmaf(sqrtf(fmaf(4.0f, e0, d1)), 1.01f, 1.0f));
}

enum { kTcTop2 = 0, kTcShortlist = 1, kTcDump = 2 };

// One 8-element group of a row: y~ = fl(x - mu), its partial ||y~||^2 (FP32
// FMA chain), and the fp16 hi/lo split of y~ * 2^ey (two elements per packed
// conversion).  bad: a value fp16 cannot hold (or NaN).  Shared by the
// in-kernel converter and the row-image builder, so both give the same bits.
__device__ __forceinline__ void tc_split8(const float (&xv)[8], const float (&mv)[8], bool valid, float sy,
                                          uint4& ph, uint4& pl, float& qq, bool& bad) {
  float yv[8];
  qq = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    yv[k] = valid ? __fsub_rn(xv[k], mv[k]) : 0.f;
    qq = fmaf(yv[k], yv[k], qq);
  }
  uint32_t hw[4], lw[4];
  float vmax = 0.f;
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const float v0 = yv[k] * sy, v1 = yv[k + 1] * sy;
    vmax = fmaxf(vmax, fmaxf(fabsf(v0), fabsf(v1)));
    const __half2 hi = __floats2half2_rn(v0, v1);
    const float2 hf = __half22float2(hi);
    const __half2 lo = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
    hw[k / 2] = *reinterpret_cast<const uint32_t*>(&hi);
    lw[k / 2] = *reinterpret_cast<const uint32_t*>(&lo);
  }
  bad = !(vmax <= 60000.0f) || isnan(qq);  // fmaxf drops NaN; the norm keeps it
  ph = make_uint4(hw[0], hw[1], hw[2], hw[3]);
  pl = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}

// Row image (rows [0, n)): item = (row, 8-element group); a row's L/8 groups
// sit in adjacent lanes and combine ||y~||^2 by shuffles in the converter's
// order, so the image equals what the converter would write.
template <int L>
__global__ void __launch_bounds__(256) build_row_image_kernel(const float* __restrict__ x32,
                                                              const float* __restrict__ mu, long long n,
                                                              float sy, unsigned short* aimg, float* aq) {
  constexpr int kG = L / 8;
  const long long items = n * kG;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long end = (items + 31) / 32 * 32;
  for (long long it0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; it0 < end; it0 += stride) {
    const bool live = it0 < items;
    const long long it = live ? it0 : 0;
    const long long row = it / kG;
    const int c8 = (int)(it % kG);
    float xv[8], mv[8];
    const float4* src = reinterpret_cast<const float4*>(x32 + row * L + c8 * 8);
    const float4 p0 = __ldg(src), p1 = __ldg(src + 1);
    xv[0] = p0.x; xv[1] = p0.y; xv[2] = p0.z; xv[3] = p0.w;
    xv[4] = p1.x; xv[5] = p1.y; xv[6] = p1.z; xv[7] = p1.w;
#pragma unroll
    for (int k = 0; k < 8; ++k) mv[k] = __ldg(mu + c8 * 8 + k);
    uint4 ph, pl;
    float qq;
    bool bb;
    tc_split8(xv, mv, live, sy, ph, pl, qq, bb);
    int bi = bb ? 1 : 0;
#pragma unroll
    for (int o = 1; o < kG; o <<= 1) {
      qq += __shfl_xor_sync(0xffffffffu, qq, o);
      bi |= __shfl_xor_sync(0xffffffffu, bi, o);
    }
    if (live) {
      const long long t = row / kTcRows;
      const int r = (int)(row % kTcRows);
      unsigned short* yh = aimg + t * (2LL * kTcRows * L);
      *reinterpret_cast<uint4*>(yh + tc_off(r, c8 * 8, L)) = ph;
      *reinterpret_cast<uint4*>(yh + kTcRows * L + tc_off(r, c8 * 8, L)) = pl;
      if (c8 == 0) aq[row] = bi ? -1.0f : qq;
    }
  }
}

cudaError_t launch_build_row_image(const float* x32, const float* mu, long long n, int dim, int ey,
                                   unsigned short* aimg, float* aq, int sms, cudaStream_t s) {
  const float sy = ldexpf(1.0f, ey);
  const int grid = sms * 8;
  switch (dim) {
    case 16: build_row_image_kernel<16><<<grid, 256, 0, s>>>(x32, mu, n, sy, aimg, aq); break;
    case 32: build_row_image_kernel<32><<<grid, 256, 0, s>>>(x32, mu, n, sy, aimg, aq); break;
    case 64: build_row_image_kernel<64><<<grid, 256, 0, s>>>(x32, mu, n, sy, aimg, aq); break;
    default: return cudaSuccess;
  }
  return cudaGetLastError();
}

// MODE kTcTop2: candidate pass over rows [r0, r1) -> idx + certified band /
//   re-rank queue (flags, flag_thr).
// MODE kTcShortlist: the queued rows again (gathered from flags): every j
//   with v_j <= thr (the same TC arithmetic, so the band argument of
//   shortlist_kernel holds with the TC error), FP64 on <= 8 candidates,
//   overflow -> flags2.  ~2 ALU ops per value instead of 5.
// MODE kTcDump: tile 0's raw accumulators -> dump (tests).
template <int L, int MODE>
__global__ void __launch_bounds__(TcCfg<L>::threads(MODE), 1) assign_tc_kernel(KernelArgs a, float* dump,
                                                                          int b_cap) {
  pdl_wait();
  using C = TcCfg<L>;
  DevState* st = a.st;
  if (pass_off(st)) return;
  const int K = st->size;
  if (MODE != kTcDump && !tc_handles(st, K)) return;
  const int ncols = K < kTcChunk ? K : kTcChunk;  // MMA N (64 / 128 for small codebooks)
  const int nch = (K + kTcChunk - 1) / kTcChunk;
  const long long nitems = MODE == kTcShortlist ? (long long)st->flag_count : a.r1 - a.r0;
  // a short queue is rescanned faster by shortlist_kernel's warp-per-row mode
  // (valid for TC-flagged rows: its FP32 error is below the TC band's)
  if (MODE == kTcShortlist && nitems * (long long)K < kTcShortlistWork) return;
  const long long ntiles = (nitems + kTcRows - 1) / kTcRows;
  const long long my_tiles = MODE == kTcDump
                                 ? 1
                                 : ((long long)blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0);
  if (my_tiles <= 0) return;

  // resident: the whole operand image sits in smem for the kernel; streaming:
  // chunks cycle through kStages slots, reloaded for every row tile
  const bool resident = nch <= b_cap;
  // rows from the prebuilt operand image (whole tiles from r0, a multiple of
  // 128; the host guarantees it) instead of the converter warps
  const bool img = MODE != kTcShortlist && a.aimg != nullptr;
  // row conversion: the converter warp, joined by the streamer warp when the
  // codebook is resident (the streamer has nothing to stream then)
  const int conv_warps = (resident ? 2 : 1) + C::kExtraConv;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sB = smem;
  unsigned char* sA = smem + (size_t)b_cap * C::kChunkBytes;
  float* sX = reinterpret_cast<float*>(sA + 2 * C::kABytes);
  using Misc = TcMisc<C::kParts>;
  static_assert(sizeof(Misc) <= C::kMisc, "misc smem");
  static_assert(offsetof(Misc, qrow) % 16 == 0, "qrow is a bulk-copy destination");
  Misc* m = reinterpret_cast<Misc*>(sA + 2 * C::kABytes + C::kXsBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // profiling builds (-DVQB_TC_PROFILE, VQB_TC_PROF=1): in kTcTop2 mode `dump`
  // collects, per warp role, the clock64 cycles spent in each barrier wait
  // and in total
#ifdef VQB_TC_PROFILE
  unsigned long long* prof = MODE == kTcTop2 ? reinterpret_cast<unsigned long long*>(dump) : nullptr;
#else
  constexpr unsigned long long* prof = nullptr;
#endif
  long long pacc[4] = {0, 0, 0, 0};
  const long long pt0 = prof ? clock64() : 0;
  auto pwait = [&](uint64_t* bar, uint32_t par, int slot) {
    if (prof) {
      const long long t = clock64();
      mbar_wait(bar, par);
      pacc[slot] += clock64() - t;
    } else {
      mbar_wait(bar, par);
    }
  };
  auto pflush = [&](int role) {
    if (prof && lane == 0) {
      pacc[3] = clock64() - pt0;
      for (int k = 0; k < 4; ++k) atomicAdd(prof + role * 4 + k, (unsigned long long)pacc[k]);
      atomicAdd(prof + 16 + role, 1ull);
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(&m->b_full, 1);
      for (int i = 0; i < C::kStages; ++i) {
        mbar_init(&m->bs_full[i], 1);
        mbar_init(&m->bs_empty[i], 1);
      }
      for (int i = 0; i < 4; ++i) mbar_init(&m->q_full[i], img ? 1 : 32 * conv_warps);
      for (int i = 0; i < 4; ++i) mbar_init(&m->xs_full[i], 1);
      for (int i = 0; i < 2; ++i) {
        mbar_init(&m->a_full[i], img ? 1 : 32 * conv_warps);
        mbar_init(&m->a_empty[i], 1);
        mbar_init(&m->d_full[i], 1);
        mbar_init(&m->d_empty[i], 32 * C::kEpiWarps);
        mbar_init(&m->res_full[i], 32 * C::kEpiWarps);
        mbar_init(&m->res_empty[i], 32 * 4);
      }
      mbar_fence_init();
    }
    __syncwarp();
    tmem_alloc(&m->tmem, 512);
  }
  // the norm term's constant A columns (0 and 1 = 2^kn) in both row buffers
  {
    const unsigned short one = __half_as_ushort(__float2half_rn(ldexpf(1.0f, st->tc_kn)));
    for (int e = threadIdx.x; e < 2 * kTcRows * 16; e += blockDim.x) {
      const int b = e / (kTcRows * 16), r = (e / 16) % kTcRows, c = e % 16;
      unsigned short* ones = reinterpret_cast<unsigned short*>(sA + b * C::kABytes) + 2 * kTcRows * L;
      ones[tc_off(r, c, 16)] = c < 2 ? one : (unsigned short)0;
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = m->tmem;

  // certification of tile i's row r from the parts' results in res[i & 1]
  // (kTcTop2; run by a certification warp, or by epilogue part 0 at L = 64)
  // loop invariants of the certification (the mbarrier waits are memory
  // clobbers: inside the lambda they would be reloaded / recomputed per tile)
  const float c_dscale = ldexpf(1.0f, st->tc_ey + st->tc_ew);
  const float c_inv = 1.0f / c_dscale;
  const float c_eyw = sqrtf((float)L) * 5.9604645e-8f * (ldexpf(1.0f, -st->tc_ey) + ldexpf(1.0f, -st->tc_ew));
  const double* const c_cb = a.cb[st->cur];
  const bool c_euclid = st->metric == kEuclidean;
  constexpr bool kHoist = L >= 32;  // at L = 16 the registers they hold cost more (K = 4096: +3 % time)
  auto certify = [&](long long i, int r) {
    const float dscale = kHoist ? c_dscale : ldexpf(1.0f, st->tc_ey + st->tc_ew);
    const float inv = kHoist ? c_inv : 1.0f / dscale;
    const float eyw = kHoist ? c_eyw
                             : sqrtf((float)L) * 5.9604645e-8f *
                                   (ldexpf(1.0f, -st->tc_ey) + ldexpf(1.0f, -st->tc_ew));
    const int rb = (int)(i & 1);
    {
      // the row's coordinates for the FP64 winner distance are fetched into
      // L1 while the tile's results are still being computed (with the
      // prebuilt row image nothing else brought them on chip)
      const long long e0 = ((long long)blockIdx.x + i * gridDim.x) * kTcRows + r;
      if (L >= 32 && e0 < nitems && MODE == kTcTop2 && a.x32 && a.dim == L) {  // (at L = 16 no gain measured)
        const char* xr = reinterpret_cast<const char*>(a.x32 + (a.r0 + e0) * L);
#pragma unroll
        for (int off = 0; off < L * 4; off += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(xr + off));
      }
    }
    if (C::kCertWarps && !prof)  // dedicated warps: sleep, do not spin
      mbar_wait_sleep(&m->res_full[rb], (uint32_t)((i >> 1) & 1), kSleepNs);
    else
      pwait(&m->res_full[rb], (uint32_t)((i >> 1) & 1), 0);
    float pm[C::kParts], p2[C::kParts];
    int pi[C::kParts];
#pragma unroll
    for (int p = 0; p < C::kParts; ++p) {
      pm[p] = m->merge.res[rb].m1[p][r];
      p2[p] = m->merge.res[rb].m2[p][r];
      pi[p] = m->merge.res[rb].i1[p][r];
    }
    const float qcur = m->merge.res[rb].q[r];
    mbar_arrive(&m->res_empty[rb]);
    const long long t = (long long)blockIdx.x + i * gridDim.x;
    const long long entry = t * kTcRows + r;
    const bool valid = entry < nitems;
    const long long row = a.r0 + entry;
    // merge the parts' exact top-2: the row's minimum M1 (first part holding
    // it), and its second minimum M2 = min(the winner part's second minimum,
    // every other part's minimum); equal minima in two parts give M2 = M1
    float M1 = pm[0], M2 = p2[0];
    int i1 = pi[0];
#pragma unroll
    for (int p = 1; p < C::kParts; ++p) {
      const bool lt = pm[p] < M1;
      M2 = fminf(lt ? p2[p] : M2, lt ? M1 : pm[p]);
      i1 = lt ? pi[p] : i1;
      M1 = lt ? pm[p] : M1;
    }
    const float E = tc_band<L>(M1 * inv, qcur, sqrtf(fmaxf(qcur, 0.f)), eyw);
    // float64 rows: + the band of their float32 rounding
    const float band = 3.0f * E + input_band(valid ? rin_of(a, row) : 0.f, M1 * inv + qcur, 3.0f * E);
    const float thr_s = fmaf(band, dscale, M1);
    // certified iff the minimum is the only value within 3E of it (see the
    // header comment and assign_chunk in kernels.cu)
    bool flag = false;
    float thr = NAN;
    if (valid) {
      flag = qcur < 0.f || !(M2 > thr_s);
      thr = M1 * inv + band;
      a.idx[row] = i1;
      if (!flag && a.dists) {
        // exact FP64 distance to the certified winner (_kernels.py:25-34);
        // the row is L2-resident from its conversion
        const double d = row_dist<L>(a, row, kHoist ? c_cb : a.cb[st->cur], i1);
        a.dists[row] = (kHoist ? c_euclid : st->metric == kEuclidean) ? sqrt(d) : d;
      }
    }
    const int lane = threadIdx.x & 31;
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
  };

  if (warp == 0) {
    // ===== MMA issuer (one thread) =====
    if (lane == 0) {
      if (resident) {
        mbar_arrive_expect_tx(&m->b_full, (uint32_t)(nch * C::kChunkBytes));
        for (int c = 0; c < nch; ++c)
          bulk_g2s(sB + c * C::kChunkBytes,
                   reinterpret_cast<const unsigned char*>(a.tcb) + (size_t)c * C::kChunkBytes,
                   (uint32_t)C::kChunkBytes, &m->b_full);
        mbar_wait(&m->b_full, 0);
        tc_fence_after();
      }
      // kind::f16 instruction descriptor: D f32, A/B f16, both K-major, N=256, M=128
      const uint32_t idesc = (1u << 4) | ((uint32_t)(ncols >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
      constexpr uint32_t kSboL = L * 16, kSbo16 = 16 * 16;
      const uint32_t sBa = smem_u32(sB), sAa = smem_u32(sA);
      long long g = 0;
      for (long long i = 0; i < my_tiles; ++i) {
        const int b = (int)(i & 1);
        pwait(&m->a_full[b], (uint32_t)((i >> 1) & 1), 0);
        tc_fence_after();
        const uint32_t aYh = sAa + b * (uint32_t)C::kABytes;
        const uint32_t aYl = aYh + kTcRows * L * 2;
        const uint32_t aOne = aYh + 2 * kTcRows * L * 2;
        for (int c = 0; c < nch; ++c, ++g) {
          const int s = (int)(g & 1);
          int stage = c;
          if (!resident) {
            stage = (int)(g % C::kStages);
            pwait(&m->bs_full[stage], (uint32_t)((g / C::kStages) & 1), 2);
          }
          pwait(&m->d_empty[s], (uint32_t)(((g >> 1) & 1) ^ 1), 1);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(s * kTcChunk);
          const uint32_t bWh = sBa + stage * (uint32_t)C::kChunkBytes;
          const uint32_t bWl = bWh + kTcChunk * L * 2;
          const uint32_t bN = bWh + 2 * kTcChunk * L * 2;
#pragma unroll
          for (int k = 0; k < L / 16; ++k) {
            const uint64_t dyh = umma_desc(aYh + k * 256, 128, kSboL);
            const uint64_t dyl = umma_desc(aYl + k * 256, 128, kSboL);
            const uint64_t dwh = umma_desc(bWh + k * 256, 128, kSboL);
            const uint64_t dwl = umma_desc(bWl + k * 256, 128, kSboL);
            mma_f16_ss(d, dyh, dwh, idesc, k > 0 ? 1u : 0u);
            mma_f16_ss(d, dyh, dwl, idesc, 1u);
            mma_f16_ss(d, dyl, dwh, idesc, 1u);
          }
          mma_f16_ss(d, umma_desc(aOne, 128, kSbo16), umma_desc(bN, 128, kSbo16), idesc, 1u);
          mma_commit(&m->d_full[s]);
          if (!resident) mma_commit(&m->bs_empty[stage]);
        }
        mma_commit(&m->a_empty[b]);
      }
    }
    pflush(0);
  } else if ((warp >= 2 + C::kEpiWarps && warp < C::kCertWarp0) || (resident && warp == 1 + C::kEpiWarps)) {
    // ===== row converters: tile i's rows -> fp16 hi/lo A buffer (i & 1) =====
    const float sy = ldexpf(1.0f, st->tc_ey);
    const int cid = warp == 1 + C::kEpiWarps ? conv_warps - 1 : warp - (2 + C::kEpiWarps);
    constexpr bool kUseXs = MODE != kTcShortlist && C::kXsBytes > 0;
    constexpr int kXs = C::kXsStages;
    auto issue_xs = [&](long long i) {  // bulk copy of tile i's contiguous rows
      const long long t = (long long)blockIdx.x + i * gridDim.x;
      const long long rows = min((long long)kTcRows, nitems - t * kTcRows);
      const uint32_t bytes = (uint32_t)(rows * L * 4);
      const int xb = (int)(i % kXs);
      mbar_arrive_expect_tx(&m->xs_full[xb], bytes);
      bulk_g2s(sX + xb * (kTcRows * L), a.xc + (a.r0 + t * kTcRows) * L, bytes, &m->xs_full[xb]);
    };
    if (img) {
      // prebuilt row image: the tile's operand rows and norms are two bulk
      // copies (no conversion work)
      if (cid == 0 && lane == 0) {
        constexpr uint32_t kImgBytes = 2u * kTcRows * L * 2u;
        for (long long i = 0; i < my_tiles; ++i) {
          const int b = (int)(i & 1);
          pwait(&m->a_empty[b], (uint32_t)(((i >> 1) & 1) ^ 1), 0);  // tile i-2's MMAs are done
          const long long tg = a.r0 / kTcRows + (long long)blockIdx.x + i * gridDim.x;
          mbar_arrive_expect_tx(&m->a_full[b], kImgBytes);
          bulk_g2s(sA + b * C::kABytes, a.aimg + tg * (2LL * kTcRows * L), kImgBytes, &m->a_full[b]);
          mbar_arrive_expect_tx(&m->q_full[i & 3], kTcRows * 4u);
          bulk_g2s(&m->qrow[i & 3][0], a.aq + tg * kTcRows, kTcRows * 4u, &m->q_full[i & 3]);
          // the certification warps read the tile's float32 rows for the FP64
          // winner distances two tiles later: bring them into L2 now (with
          // the image nothing else touches x32, and that HBM round trip per
          // tile bounded the single-chunk passes)
          if (L >= 32 && MODE == kTcTop2 && a.x32 && a.dim == L && a.dists) {  // (at L = 16: +1 % time)
            const long long row0 = tg * kTcRows;
            const long long rows = min((long long)kTcRows, a.n - row0);
            if (rows > 0) bulk_prefetch_l2(a.x32 + row0 * L, (uint32_t)(rows * L * 4));
          }
        }
      }
    } else {
    if (kUseXs && cid == 0 && lane == 0)
      for (int j = 0; j < kXs && j < my_tiles; ++j) issue_xs(j);
    // the centring vector, in registers for the whole kernel (L <= 32)
    constexpr int kMuRegs = L <= 32 ? L : 1;
    float mur[kMuRegs];
#pragma unroll
    for (int k = 0; k < kMuRegs; ++k) mur[k] = a.mu[k];
    for (long long i = 0; i < my_tiles; ++i) {
      const int b = (int)(i & 1);
      pwait(&m->a_empty[b], (uint32_t)(((i >> 1) & 1) ^ 1), 0);  // tile i-2's MMAs are done
      const float* xs = sX + (int)(i % kXs) * (kTcRows * L);
      if (kUseXs) pwait(&m->xs_full[i % kXs], (uint32_t)((i / kXs) & 1), 1);
      unsigned short* yh = reinterpret_cast<unsigned short*>(sA + b * C::kABytes);
      unsigned short* yl = yh + kTcRows * L;
      const long long t = (long long)blockIdx.x + i * gridDim.x;
      // work item = (row, 8-element group): independent items give the
      // converter ILP; a row's L/8 groups sit in adjacent lanes and combine
      // ||y~||^2 by shuffles (whole warps iterate: items past the tile idle)
      constexpr int kG = L / 8;
      const int it_end = (kTcRows * kG + 32 * conv_warps - 1) / (32 * conv_warps) * (32 * conv_warps);
#pragma unroll 4
      for (int it0 = cid * 32 + lane; it0 < it_end; it0 += 32 * conv_warps) {
        const bool live = it0 < kTcRows * kG;
        const int it = live ? it0 : 0;
        const int r = it / kG, c8 = it % kG;
        const long long entry = t * kTcRows + r;
        const bool valid = live && entry < nitems;
        const long long row = MODE == kTcShortlist ? (valid ? (long long)a.flags[entry] : 0) : a.r0 + entry;
        float xv[8], mv[8];
        if (valid) {
          const float4* src = kUseXs ? reinterpret_cast<const float4*>(xs + r * L + c8 * 8)
                                     : reinterpret_cast<const float4*>(a.xc + row * L + c8 * 8);
          const float4 p0 = kUseXs ? src[0] : __ldg(src), p1 = kUseXs ? src[1] : __ldg(src + 1);
          xv[0] = p0.x; xv[1] = p0.y; xv[2] = p0.z; xv[3] = p0.w;
          xv[4] = p1.x; xv[5] = p1.y; xv[6] = p1.z; xv[7] = p1.w;
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) xv[k] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if constexpr (L <= 32) {
            mv[k] = mur[k % kMuRegs];
#pragma unroll
            for (int g = 1; g < kG; ++g) mv[k] = c8 == g ? mur[(g * 8 + k) % kMuRegs] : mv[k];
          } else {
            mv[k] = __ldg(a.mu + c8 * 8 + k);
          }
        }
        uint4 ph, pl;
        float qq;
        bool bb;
        tc_split8(xv, mv, valid, sy, ph, pl, qq, bb);
        if (live) {
          *reinterpret_cast<uint4*>(yh + tc_off(r, c8 * 8, L)) = ph;
          *reinterpret_cast<uint4*>(yl + tc_off(r, c8 * 8, L)) = pl;
        }
        int bi = bb ? 1 : 0;
#pragma unroll
        for (int o = 1; o < kG; o <<= 1) {
          qq += __shfl_xor_sync(0xffffffffu, qq, o);
          bi |= __shfl_xor_sync(0xffffffffu, bi, o);
        }
        if (live && c8 == 0) m->qrow[i & 3][r] = bi ? -1.0f : qq;
      }
      if (kUseXs) {
        // every converter lane is done with the stage: fetch the next tile
        if (conv_warps > 1) named_bar(4, 32 * conv_warps); else __syncwarp();
        if (cid == 0 && lane == 0 && i + kXs < my_tiles) issue_xs(i + kXs);
      }
      fence_proxy_async_smem();
      mbar_arrive(&m->a_full[b]);
      mbar_arrive(&m->q_full[i & 3]);
    }
    }
    pflush(1);
  } else if (warp == 1 + C::kEpiWarps) {
    // ===== codebook streamer (streaming mode only) =====
    if (!resident && lane == 0) {
      long long g = 0;
      for (long long i = 0; i < my_tiles; ++i) {
        for (int c = 0; c < nch; ++c, ++g) {
          const int stage = (int)(g % C::kStages);
          mbar_wait(&m->bs_empty[stage], (uint32_t)(((g / C::kStages) & 1) ^ 1));
          mbar_arrive_expect_tx(&m->bs_full[stage], (uint32_t)C::kChunkBytes);
          bulk_g2s(sB + stage * C::kChunkBytes,
                   reinterpret_cast<const unsigned char*>(a.tcb) + (size_t)c * C::kChunkBytes,
                   (uint32_t)C::kChunkBytes, &m->bs_full[stage]);
        }
      }
    }
  } else if (warp >= C::kCertWarp0) {
    // ===== certification warps (kTcTop2): lane = row of the tile quarter =====
    if constexpr (MODE == kTcTop2)
      for (long long i = (warp - C::kCertWarp0) >> 2; i < my_tiles; i += C::kCertGroups)
        certify(i, ((warp - C::kCertWarp0) & 3) * 32 + lane);
    pflush(3);
  } else {
    // ===== epilogue warps: row conversion + per-value work over TMEM =====
    const int e = warp - 1;
    const int h = e >> 2;       // column part of every 256-column chunk (0: owns the row)
    const int qd = warp & 3;    // TMEM lane quarter this warp may access
    const int r = qd * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const float sy = ldexpf(1.0f, st->tc_ey);
    const float dscale = ldexpf(1.0f, st->tc_ey + st->tc_ew);

    // row of (local tile i, tile row r); valid = inside the range / queue
    auto row_of = [&](long long i, long long& entry, bool& valid) -> long long {
      const long long t = (long long)blockIdx.x + i * gridDim.x;
      entry = t * kTcRows + r;
      valid = entry < nitems;
      if (MODE == kTcShortlist) return valid ? (long long)a.flags[entry] : 0;
      return a.r0 + entry;
    };

    auto min16 = [](const float* v) {
      const float t0 = fminf(fminf(v[0], v[1]), v[2]), t1 = fminf(fminf(v[3], v[4]), v[5]);
      const float t2 = fminf(fminf(v[6], v[7]), v[8]), t3 = fminf(fminf(v[9], v[10]), v[11]);
      const float t4 = fminf(fminf(v[12], v[13]), v[14]);
      return fminf(fminf(fminf(t0, t1), t2), fminf(fminf(t3, t4), v[15]));
    };
    long long g = 0;
    for (long long i = 0; i < my_tiles; ++i) {
      // kTcTop2: running top-2 of the block minima (b1, b2; blk = first block
      // at b1) and the 16 class chains; kTcShortlist: candidate list
      float b1 = INFINITY, b2 = INFINITY;
      int blk = 0;
      float ach[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) ach[t] = INFINITY;
      int nc = 0;
      int cand[kTcShort] = {0, 0, 0, 0, 0, 0, 0, 0};
      float thr_d = -INFINITY;
      long long entry;
      bool valid;
      const long long row = row_of(i, entry, valid);
      if (MODE == kTcShortlist && valid) thr_d = a.flag_thr[entry] * dscale;  // NaN stays NaN -> overflow
      float qcur = 0.f;
      if constexpr (MODE == kTcTop2) {
        if (h == 0) {
          pwait(&m->q_full[i & 3], (uint32_t)((i >> 2) & 1), 0);
          qcur = m->qrow[i & 3][r];
        }
      }
      for (int c = 0; c < nch; ++c, ++g) {
        const int s = (int)(g & 1);
        pwait(&m->d_full[s], (uint32_t)((g >> 1) & 1), 1);
        tc_fence_after();
        const int span = ncols / C::kParts;  // this part's columns of the chunk
        // 32 accumulator columns of this part (padded with +inf below 32)
        auto load = [&](int q4, float (&v)[32]) {
          const int col = s * kTcChunk + h * span + q4 * 32;
          if (span >= 32) {
            tmem_ld32(trow + (uint32_t)col, v);
          } else {
            float v16[16];
            tmem_ld16(trow + (uint32_t)col, v16);
#pragma unroll
            for (int t = 0; t < 16; ++t) v[t] = v16[t];
#pragma unroll
            for (int t = 16; t < 32; ++t) v[t] = INFINITY;  // never a candidate
          }
          tmem_wait_ld();
        };
        if constexpr (MODE == kTcTop2) {
          // ONE read of the chunk, exact top-2 by minima only (half a 3-input
          // FMNMX per value and partition, no per-value compare): the values
          // of a part are covered by two partitions -- 16 persistent chains
          // by column mod 16 (A) and blocks of 16 consecutive columns (B,
          // folded into a running top-2 of the block minima).  Any two
          // columns differ in class or in block, so the row's second minimum
          // is min(second smallest A chain, second smallest block minimum);
          // its minimum is at (first block holding it) + (class holding it).
          const uint32_t cbase = trow + (uint32_t)(s * kTcChunk + h * span);
          const int jb0 = c * kTcChunk + h * span;
          auto fold = [&](float mu, int jb) {  // block minimum into the running top-2
            const bool lt = mu < b1;
            b2 = fminf(b2, fmaxf(b1, mu));
            b1 = fminf(b1, mu);
            blk = lt ? jb : blk;
          };
          auto scan32 = [&](const float (&v)[32], int q4) {
#pragma unroll
            for (int t = 0; t < 16; ++t) ach[t] = fminf(fminf(v[t], v[t + 16]), ach[t]);
            // both block minima in one step: the pair sorted (lo <= hi), then
            // the two smallest of {b1, b2, lo, hi} = min(b1, lo) and
            // min3(b2, hi, max(b1, lo)) -- one half-rate FMNMX less than two
            // single folds; the first block at the minimum keeps its index
            // (lo < b1 strictly, and block 0 on mu0 == mu1)
            const float mu0 = min16(v), mu1 = min16(v + 16);
            const int jb = jb0 + q4 * 32;
            const float lo = fminf(mu0, mu1), hi = fmaxf(mu0, mu1);
            const int jlo = mu1 < mu0 ? jb + 16 : jb;
            const bool lt = lo < b1;
            b2 = fminf(fminf(b2, hi), fmaxf(b1, lo));
            b1 = fminf(b1, lo);
            blk = lt ? jlo : blk;
          };
          if (span >= 32) {
            if (pipe_ld<L>() && span >= 64) {
              // 8 epilogue warps (2 per scheduler): the load of group g + 1 is
              // in flight while group g is scanned (two register buffers)
              const int ng = span / 32;
              float va[32], vb[32];
              tmem_ld32(cbase, va);
#pragma unroll 1
              for (int q4 = 0; q4 < ng; q4 += 2) {
                tmem_wait_ld();
                if (q4 + 1 < ng) tmem_ld32(cbase + (uint32_t)((q4 + 1) * 32), vb);
                scan32(va, q4);
                if (q4 + 1 < ng) {
                  tmem_wait_ld();
                  if (q4 + 2 < ng) tmem_ld32(cbase + (uint32_t)((q4 + 2) * 32), va);
                  scan32(vb, q4 + 1);
                }
              }
            } else {
#pragma unroll 1
              for (int q4 = 0; q4 < span / 32; ++q4) {
                float v[32];
                tmem_ld32(cbase + (uint32_t)(q4 * 32), v);
                tmem_wait_ld();
                scan32(v, q4);
              }
            }
          } else {
            float v[16];
            tmem_ld16(cbase, v);
            tmem_wait_ld();
#pragma unroll
            for (int t = 0; t < 16; ++t) ach[t] = fminf(v[t], ach[t]);
            fold(min16(v), jb0);
          }
        } else {
#pragma unroll 1
          for (int q4 = 0; q4 < (span + 31) / 32; ++q4) {
            float v[32];
            load(q4, v);
            const int jb = c * kTcChunk + h * span + q4 * 32;
            if constexpr (MODE == kTcDump) {
#pragma unroll
              for (int t = 0; t < 32; ++t)
                if (t < span) dump[(long long)r * K + jb + t] = v[t];
            } else {
              // hit mask of the group (FSETP + predicated OR per value; the
              // +inf padding and columns past K never hit), then the few hits
              // are appended through a select network so the candidate list
              // stays in registers (a dynamically indexed array would live in
              // local memory)
              unsigned msk = 0u;
#pragma unroll
              for (int t = 0; t < 32; ++t)
                asm("{\n\t.reg .pred p;\n\tsetp.le.f32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}"
                    : "+r"(msk)
                    : "f"(v[t]), "f"(thr_d), "r"(1u << t));
              while (msk) {
                const int jt = jb + __ffs(msk) - 1;
                msk &= msk - 1u;
#pragma unroll
                for (int k = 0; k < kTcShort; ++k) cand[k] = nc == k ? jt : cand[k];
                ++nc;
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&m->d_empty[s]);
      }
      if constexpr (MODE == kTcTop2) {
        // hand the tile's per-part results to the certification warps
        // the part's top-2: the chains' second smallest (as a multiset: two
        // classes at the minimum give s2 = s1) and the class of the minimum
        // The chains' minimum is b1 itself (both are the minimum of the part's
        // values), so: mark the chains equal to b1 (one FSETP each, feeding a
        // predicated OR into the mask and the select that takes the chain out
        // of the second-minimum tree); cls = the first marked chain; two
        // marked chains make the second minimum b1.
        unsigned eqm = 0u;
        float rest[16];
#pragma unroll
        for (int t = 0; t < 16; ++t)
          asm("{\n\t.reg .pred p;\n\tsetp.eq.f32 p, %2, %3;\n\t@p or.b32 %0, %0, %4;\n\t"
              "selp.f32 %1, 0f7F800000, %2, p;\n\t}"
              : "+r"(eqm), "=f"(rest[t])
              : "f"(ach[t]), "f"(b1), "r"(1u << t));
        const int cls = eqm ? __ffs(eqm) - 1 : 0;
        const float s2 = (eqm & (eqm - 1u)) ? b1 : min16(rest);
        const int rb = (int)(i & 1);
        pwait(&m->res_empty[rb], (uint32_t)(((i >> 1) & 1) ^ 1), 2);
        m->merge.res[rb].m1[h][r] = b1;
        m->merge.res[rb].m2[h][r] = fminf(b2, s2);
        m->merge.res[rb].i1[h][r] = blk + cls;
        if (h == 0) m->merge.res[rb].q[r] = qcur;
        mbar_arrive(&m->res_full[rb]);
        if (!C::kCertWarps && h == 0) certify(i, r);
      } else if constexpr (MODE == kTcShortlist) {
        // every part evaluates its own candidates in FP64 (a part holding more
        // than kTcShort, or a row out of fp16 range, overflows the row anyway);
        // one barrier, then part 0 decides overflow from the total and merges
        // the parts' lexicographic minima.  The merge area alternates by tile
        // parity: part 0 has finished reading area (i & 1) before it reaches
        // tile i + 1's barrier, which every part passes before writing tile
        // i + 2 into the same area.
        auto& ml = m->merge.sl[i & 1];
        ml.count[h][r] = (unsigned char)min(nc, 255);
        mbar_wait(&m->q_full[i & 3], (uint32_t)((i >> 2) & 1));
        const bool bad = m->qrow[i & 3][r] < 0.f;
        double best = INFINITY;
        int bj = 0x7fffffff;
        if (valid && !bad && nc <= kTcShort) {
          // the reference's arithmetic (_kernels.py:25-29); (d, j) order
          const double* __restrict__ cb = a.cb[st->cur];
#pragma unroll
          for (int k = 0; k < kTcShort; ++k) {  // unrolled: cand[] stays in registers
            if (k < nc) {
              const double d = row_dist<L>(a, row, cb, cand[k]);
              if (d < best || (d == best && cand[k] < bj)) {
                best = d;
                bj = cand[k];
              }
            }
          }
        }
        ml.best[h][r] = best;
        ml.bestj[h][r] = bj;
        named_bar(2, 32 * C::kEpiWarps);
        if (h == 0 && valid) {
          int total = 0;
#pragma unroll
          for (int p = 0; p < C::kParts; ++p) total += ml.count[p][r];
          const bool over = total == 0 || total > kTcShort || bad;
          if (over) {
            const int pos = atomicAdd(&st->flag2_count, 1);
            a.flags2[pos] = (int)row;
          } else {
#pragma unroll
            for (int p = 1; p < C::kParts; ++p) {
              const double d = ml.best[p][r];
              const int j = ml.bestj[p][r];
              if (d < best || (d == best && j < bj)) {
                best = d;
                bj = j;
              }
            }
            a.idx[row] = (best < INFINITY) ? bj : 0;  // nothing < inf -> index 0
            if (a.dists) a.dists[row] = st->metric == kEuclidean ? sqrt(best) : best;
          }
        }
      }
    }
    pflush(2);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int L, int MODE>
static cudaError_t launch_tc_L(const KernelArgs& a, int grid, float* dump, cudaStream_t s) {
  using C = TcCfg<L>;
  const long long kchunks = (a.kmax + kTcChunk - 1) / kTcChunk;
  if (kchunks < 1 || !a.tcb) return cudaSuccess;
  // B region: the whole image when it fits (resident), else the ring
  const int b_cap = (int)(kchunks <= C::kMaxChunks ? kchunks : C::kMaxChunks);
  const size_t smem =
      (size_t)std::max(b_cap, C::kStages) * C::kChunkBytes + 2 * C::kABytes + C::kXsBytes + C::kMisc;
  cudaError_t e = cudaFuncSetAttribute(assign_tc_kernel<L, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  {
    cudaError_t e1 = launch_k(assign_tc_kernel<L, MODE>, grid, C::threads(MODE), smem, s, a, dump, b_cap);
    if (e1 != cudaSuccess) return e1;
  }
  return cudaGetLastError();
}

// VQB_TC_PROF=1 (tools only): per warp role, the share of the kernel's
// cycles each role spends in its barrier waits, printed to stderr after every
// launch (synchronises the stream)
static unsigned long long* tc_prof_buffer() {
#ifndef VQB_TC_PROFILE
  return nullptr;
#endif
  static unsigned long long* buf = nullptr;
  static const bool on = [] {
    const char* e = std::getenv("VQB_TC_PROF");
    return e && e[0] == '1';
  }();
  if (on && !buf && cudaMalloc(&buf, 32 * sizeof(unsigned long long)) != cudaSuccess) buf = nullptr;
  return on ? buf : nullptr;
}

cudaError_t launch_assign_tc(const KernelArgs& a_in, int sms, cudaStream_t s) {
  KernelArgs a = a_in;
  if (a.r0 % kTcRows != 0) a.aimg = nullptr;  // the image is tiled from row 0
  unsigned long long* prof = tc_prof_buffer();
  if (prof) cudaMemsetAsync(prof, 0, 32 * sizeof(unsigned long long), s);
  float* pd = reinterpret_cast<float*>(prof);
  cudaError_t e = cudaSuccess;
  switch (a.cdim) {
    case 16: e = launch_tc_L<16, kTcTop2>(a, sms, pd, s); break;
    case 32: e = launch_tc_L<32, kTcTop2>(a, sms, pd, s); break;
    case 64: e = launch_tc_L<64, kTcTop2>(a, sms, pd, s); break;
    default: return cudaSuccess;
  }
  if (prof && e == cudaSuccess) {
    unsigned long long h[32];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    static const char* role[4] = {"mma", "conv", "epi", "cert"};
    static const char* slot[4][3] = {{"a_full", "d_empty", "bs_full"},
                                     {"a_empty", "xs_full", "-"},
                                     {"q_full", "d_full", "res_empty"},
                                     {"res_full", "-", "-"}};
    for (int r = 0; r < 4; ++r) {
      if (!h[16 + r] || !h[r * 4 + 3]) continue;
      std::fprintf(stderr, "tcprof %s warps=%llu", role[r], h[16 + r]);
      for (int k = 0; k < 3; ++k)
        std::fprintf(stderr, " %s=%.3f", slot[r][k], (double)h[r * 4 + k] / (double)h[r * 4 + 3]);
      std::fprintf(stderr, " cycles/warp=%.0f\n", (double)h[r * 4 + 3] / (double)h[16 + r]);
    }
  }
  return e;
}

cudaError_t launch_shortlist_tc(const KernelArgs& a, int sms, cudaStream_t s) {
  switch (a.cdim) {
    case 16: return launch_tc_L<16, kTcShortlist>(a, sms, nullptr, s);
    case 32: return launch_tc_L<32, kTcShortlist>(a, sms, nullptr, s);
    case 64: return launch_tc_L<64, kTcShortlist>(a, sms, nullptr, s);
    default: return cudaSuccess;
  }
}

cudaError_t launch_tc_probe(const KernelArgs& a, float* dump, cudaStream_t s) {
  switch (a.cdim) {
    case 16: return launch_tc_L<16, kTcDump>(a, 1, dump, s);
    case 32: return launch_tc_L<32, kTcDump>(a, 1, dump, s);
    case 64: return launch_tc_L<64, kTcDump>(a, 1, dump, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vqb
