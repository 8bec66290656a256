// fp64 Gram X_i^T X_i of the Gram path on the int8 tensor cores.
//
// The one-time G_i = Xhat_i^T Xhat_i (V_i x T, fp64) is computed from exact
// int8 slices of Xhat (an Ozaki-style splitting with a power-of-two scale per
// column t):
//
//   x[v][t] = 2^{e_t} * sum_s q_s[v][t] 2^{-6-7s} + r,   |q_s| <= 64,
//   |r| <= 2^{e_t} 2^{-7S-6} / 2,
//
// where 2^{e_t} >= max_v |x[v][t]|.  Then
//
//   G[a][b] ~= 2^{e_a+e_b} sum_{d=0}^{S-1} 2^{-12-7d} sum_{s+s'=d} (Q_s^T Q_s')[a][b]
//
// Every inner product of int8 slices is exact in int32 (|q| <= 64, at most
// S pairs per d, at most kOzChunkBlocks * 32 voxels per accumulation), so the
// only approximations are the truncation of x to 6 + 7 (S - 1) bits below its
// column maximum and the dropped pairs s + s' >= S: with S = 7 each product
// x_a x_b is represented to ~2^-48 of 2^{e_a+e_b}, ~1e-14 relative to G for
// data with column max/rms ~ 5 (BASELINE recipe).  The fp64 result then feeds
// the same per-iteration B = S G / 2 as the fp64 DMMA Gram.
//
// Kernels (the column maxima max |x[:, t]| come from the demean pass, k_prep):
//   oz_split   slices, transposed: Q[i][t][vb][slot][32 voxels] (int8; a
//              256-byte record per (t, 32-voxel block): slices 0-3 in the low
//              128 bytes, 4-6 (+ an unused slot) in the high 128 bytes; fp32
//              X-hat: four slices in 128-byte records)
//   oz_gram    one 128 x 128 upper tile per CTA: TMA (SWIZZLE_128B, 128-byte
//              rows) -> tcgen05.mma kind::i8 (M = N = 128, K = 32 voxels; the
//              slice is selected by the 32-byte descriptor advance) -> four
//              int32 accumulators in TMEM (512 columns).  Pass 1 accumulates
//              d = 0..3 from the low halves, pass 2 d = 4..6 from both halves
//              (four-slice data: the low halves again, all 16 pairs); the
//              epilogue warps scale and sum the d-groups in fp64 in order.
#include <cuda.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "plan.h"
#include "tcgen05.cuh"

namespace srm {

namespace {

using namespace tc;

constexpr int kOzSlices = 7;
constexpr int kOzThreads = 320;  // warp 0 TMA producer, warp 1 MMA issuer, warps 2-9 epilogue
constexpr int kOzStages = 3;
constexpr int kOzBox = 16384;    // one 128-row x 128-byte SW128 box
constexpr int kOzStageBytes = 4 * kOzBox;

// 2^e as a double for the normal range (|e| < 1023): exact scale factors for the
// d-group sums and the column/row exponents (a multiply, not an ldexp call)
__device__ __forceinline__ double pow2(int e) {
  return (e >= -1022 && e <= 1023) ? __longlong_as_double((long long)(1023 + e) << 52) : ldexp(1.0, e);
}

__device__ __forceinline__ int frexp_exp(double m) {
  int e = 0;
  frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  return e;
}

// ---------------------------------------------------------------------------
// split: grid (32-voxel blocks, 64-column tiles, subjects); thread (t, quarter)
// handles 8 voxels of one column, 4 voxels per packed 32-bit word.  The
// slicing of later subjects is enqueued beside the Gram of earlier ones, but
// its CTAs do not share an SM with a resident k_oz_gram CTA: three of that
// CTA's ten warps x 168 registers fill a sub-partition's 16,384, and its 195 KB
// take the 196 KB carve-out (tools/coresidency_probe.cu; session-6 entries of
// profiles/r2s3/rejected_experiments.md).  It runs on the SMs the Gram's
// one-wave batches leave free and in the gaps between batches.
// ---------------------------------------------------------------------------
constexpr int kSplitCols = 64;
constexpr int kSplitGroups = 8;  // voxel-block groups per k_oz_split CTA (fp64 X-hat)
constexpr int kSplitLdw = 68;  // words per smem row: 16-byte aligned, conflict-free uint4 access

// rint(y) for |y| < 2^51 by the 1.5 * 2^52 shift; the rounded integer is also
// the low word of the shifted value (two's complement), so no F2I is needed
__device__ __forceinline__ double round_shift(double y, int* low) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  const double t = y + magic;
  *low = __double2loint(t);
  return t - magic;
}

// nsl slices per value (7 for fp64 X-hat, 4 for fp32); records of `rec` bytes
// (256: eight 32-voxel slots; 128: four), slots beyond nsl zero.  NB
// consecutive 32-voxel blocks per CTA, so every column's records go out as one
// contiguous NB x rec-byte run (fp32's 128-byte records alone are too short a
// DRAM burst at the lq stride between columns: 0.35 of HBM with NB = 1)
//
// A CTA walks `gsz` consecutive groups of NB voxel blocks of its 64 columns,
// the next group's values loaded into registers ahead of the current group's
// arithmetic (one-group CTAs spent most of their ~3 us on launch and load
// latency): 3.85 -> 3.35 ms on cfg 2, 0.90 of the measured HBM copy rate.
template <typename TX, int NSL, int NB>
__global__ void __launch_bounds__(256) k_oz_split(DevPlan p, const TX* __restrict__ xhat, int64_t ldsrc, int64_t ncols,
                                                  const unsigned long long* __restrict__ cmax,
                                                  int8_t* __restrict__ q, int64_t lq, int32_t* __restrict__ expo,
                                                  int gsz) {
  constexpr int nsl = NSL;
  constexpr int rec = NSL <= 4 ? 128 : 256;
  static_assert(NB * rec <= 256, "a column's NB records must fit one shared-memory row");
  __shared__ __align__(16) uint32_t buf[kSplitCols * kSplitLdw];
  const int i = blockIdx.z;
  const int64_t* sj = p.subj + (int64_t)i * kSubjCols;
  const int64_t row0 = sj[SC_ROW_OFF], V = sj[SC_V];
  const int64_t vb_first = (int64_t)blockIdx.x * NB * gsz;
  if (vb_first * 32 >= V) return;
  const int64_t t0 = (int64_t)blockIdx.y * kSplitCols;
  const int tl = threadIdx.x & (kSplitCols - 1), quarter = threadIdx.x / kSplitCols;
  const int64_t t = t0 + tl;
  const bool tin = t < ncols;
  int e = 0;
  if (tin) {
    const double m = __longlong_as_double((long long)cmax[(int64_t)i * ncols + t]);
    e = (m > 0.0) ? frexp_exp(m) : 0;
    if (vb_first == 0 && quarter == 0) expo[(int64_t)i * ncols + t] = e;
  }
  TX xv[NB][8], xn[NB][8];
  auto load_group = [&](TX (&x)[NB][8], int64_t vb) {
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t v = (vb + j) * 32 + quarter * 8 + u;
        x[j][u] = (tin && v < V) ? xhat[(row0 + v) * ldsrc + t] : TX(0);
      }
  };
  load_group(xv, vb_first);
  uint2* row = reinterpret_cast<uint2*>(buf + tl * kSplitLdw);
  const int nslot = rec / 32;
  for (int gi = 0; gi < gsz; ++gi) {
  const int64_t vb0 = vb_first + (int64_t)gi * NB;
  if (vb0 * 32 >= V) break;  // (uniform over the CTA)
  const int nb = (int)min((int64_t)NB, (V + 31) / 32 - vb0);  // blocks of this subject in the group
  const bool more = gi + 1 < gsz && (vb0 + NB) * 32 < V;
  if (more) load_group(xn, vb0 + NB);
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    uint32_t w[NSL][2];
#pragma unroll
    for (int s = 0; s < NSL; ++s)
#pragma unroll
      for (int g = 0; g < 2; ++g) w[s][g] = 0u;
    // y = x 2^(6 - e), |y| < 64; digit s = rint(y), then y = (y - rint(y)) * 128.
    // Every step is exact in the input's own precision, so fp32 X-hat slices in
    // fp32 arithmetic (twice the fp64 rate) with the same digits as in fp64.
    bool done = false;
    if constexpr (sizeof(TX) == 4) {
      if (e >= -120 && e <= 130) {  // 2^(6 - e) is a normal float
        const float scale = __int_as_float((127 + 6 - e) << 23);
        const float magic = 12582912.0f;  // 1.5 * 2^23: rint for |y| < 2^22, low byte = digit
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float y = xv[j][u] * scale;
#pragma unroll
          for (int s = 0; s < NSL; ++s) {
            const float tt = y + magic;
            w[s][u >> 2] |= (uint32_t)(__float_as_int(tt) & 0xFF) << (8 * (u & 3));
            y = (y - (tt - magic)) * 128.0f;
          }
        }
        done = true;
      }
    }
    if (!done) {
      // 2^(6 - e) exactly (normal range: |e| < 1000)
      const double scale = __longlong_as_double((long long)(1023 + 6 - e) << 52);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        double y = to_f64(xv[j][u]) * scale;  // |y| < 64
#pragma unroll
        for (int s = 0; s < NSL; ++s) {
          int low;
          const double r = round_shift(y, &low);
          w[s][u >> 2] |= (uint32_t)(low & 0xFF) << (8 * (u & 3));
          y = (y - r) * 128.0;  // exact: |y - r| <= 1/2
        }
      }
    }
    // record layout per t: slot s = 8 words (32 voxels), this quarter's 8 voxels
    // at words 2 quarter, 2 quarter + 1 (slots >= nsl: zero in smem, not stored);
    // block j's record at byte j * rec of the column's row
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (s < nslot) row[j * (rec / 8) + s * 4 + quarter] = (s < nsl) ? make_uint2(w[s][0], w[s][1]) : make_uint2(0u, 0u);
  }
  __syncthreads();
  // kSplitCols rows x nb x rec / 16 chunks of 16 bytes; consecutive threads write
  // one column's run.  Slot 7 of a seven-slice record is never read by an MMA:
  // not written (NB = 1 there).
  const int nch = nsl == 7 ? 14 : nb * rec / 16;
  for (int c = threadIdx.x; c < kSplitCols * nch; c += blockDim.x) {
    const int r = c / nch, k = c % nch;
    const int64_t tt = t0 + r;
    if (tt < ncols) {
      uint4* dst = reinterpret_cast<uint4*>(q + ((int64_t)i * ncols + tt) * lq + vb0 * rec);
      dst[k] = reinterpret_cast<const uint4*>(buf + r * kSplitLdw)[k];
    }
  }
  if (!more) break;
  __syncthreads();  // the staged rows are out: the next group may overwrite them
#pragma unroll
  for (int j = 0; j < NB; ++j)
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[j][u] = xn[j][u];
  }
}

// fp32 X-hat: the four slices from one integer per value.  N = rint(x 2^(27-e))
// (|N| <= 2^27; the same 2^-27-of-the-column-max truncation as the digit
// recurrence above) is cut into balanced base-128 digits, least significant
// first: d = sext7(N), N = (N - d) >> 7 -- integer ops instead of a float
// round/subtract/scale chain per digit, and four voxels' digits are packed
// with byte permutes.  The reconstructed value sum_s q_s 2^{-7s} equals the
// recurrence's except for which way an exact tie rounds.  Full tiles (the
// common case) skip the per-value bounds checks.
template <int NB>
__global__ void __launch_bounds__(256) k_oz_split_f32(DevPlan p, const float* __restrict__ xhat,
                                                      const unsigned long long* __restrict__ cmax,
                                                      int8_t* __restrict__ q, int64_t lq, int32_t* __restrict__ expo) {
  constexpr int rec = 128;
  constexpr int LDW = NB * rec / 4 + 4;  // words per column row: NB records + 16 B (16-byte aligned)
  __shared__ __align__(16) uint32_t buf[kSplitCols * LDW];
  const int i = blockIdx.z;
  const int64_t* sj = p.subj + (int64_t)i * kSubjCols;
  const int64_t row0 = sj[SC_ROW_OFF], V = sj[SC_V];
  const int64_t vb0 = (int64_t)blockIdx.x * NB;
  if (vb0 * 32 >= V) return;
  const int64_t ldx = p.ldx;
  const int nb = (int)min((int64_t)NB, (V + 31) / 32 - vb0);
  const int64_t t0 = (int64_t)blockIdx.y * kSplitCols;
  const int tl = threadIdx.x & (kSplitCols - 1), quarter = threadIdx.x / kSplitCols;
  const int64_t t = t0 + tl;
  const bool tin = t < ldx;
  int e = 0;
  if (tin) {
    const double m = __longlong_as_double((long long)cmax[(int64_t)i * ldx + t]);
    e = (m > 0.0) ? frexp_exp(m) : 0;
    if (vb0 == 0 && quarter == 0) expo[(int64_t)i * ldx + t] = e;
  }
  float xv[NB][8];
  const float* px = xhat + (row0 + vb0 * 32 + quarter * 8) * ldx + t;
  if (tin && (vb0 + NB) * 32 <= V) {
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[j][u] = px[(int64_t)(j * 32 + u) * ldx];
  } else {
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t v = (vb0 + j) * 32 + quarter * 8 + u;
        xv[j][u] = (tin && v < V) ? px[(int64_t)(j * 32 + u) * ldx] : 0.f;
      }
  }
  // N = rint(x 2^(27 - e)): the scale as a float when it is a normal one
  // (|e| of any fp32 column maximum short of the tiny / huge extremes), else fp64
  int nv[NB][8];
  if (e >= -100 && e <= 153) {
    const float sf = __int_as_float((127 + 27 - e) << 23);
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int u = 0; u < 8; ++u) nv[j][u] = __float2int_rn(xv[j][u] * sf);
  } else {
    const double sd = ldexp(1.0, 27 - e);
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
      for (int u = 0; u < 8; ++u) nv[j][u] = __double2int_rn((double)xv[j][u] * sd);
  }
  uint2* row = reinterpret_cast<uint2*>(buf + tl * LDW);
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    int dg[4][8];  // [slice][voxel]
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      // balanced base-128 digits, least significant first: with n' = (n + 64) >> 7
      // the digit n - 128 n' lies in [-64, 63]
      int n = nv[j][u];
#pragma unroll
      for (int sl = 3; sl >= 1; --sl) {
        const int n1 = (n + 64) >> 7;
        dg[sl][u] = n - (n1 << 7);
        n = n1;
      }
      dg[0][u] = n;  // |n| <= 64
    }
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
      uint32_t w[2];
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const uint32_t lo = __byte_perm((uint32_t)dg[sl][4 * g], (uint32_t)dg[sl][4 * g + 1], 0x0040);
        const uint32_t hi = __byte_perm((uint32_t)dg[sl][4 * g + 2], (uint32_t)dg[sl][4 * g + 3], 0x0040);
        w[g] = __byte_perm(lo, hi, 0x5410);
      }
      row[j * (rec / 8) + sl * 4 + quarter] = make_uint2(w[0], w[1]);
    }
  }
  __syncthreads();
  const int nch = nb * rec / 16;
  for (int c = threadIdx.x; c < kSplitCols * nch; c += blockDim.x) {
    const int r = c / nch, k = c - r * nch;
    const int64_t tt = t0 + r;
    if (tt < ldx) {
      uint4* dst = reinterpret_cast<uint4*>(q + ((int64_t)i * ldx + tt) * lq + vb0 * rec);
      dst[k] = reinterpret_cast<const uint4*>(buf + r * LDW)[k];
    }
  }
}

// ---------------------------------------------------------------------------
// gram tiles
// ---------------------------------------------------------------------------
struct OzBars {
  uint64_t full[kOzStages];
  uint64_t empty[kOzStages];
  uint64_t accfull;
  uint64_t accfree;
};

// descriptor address-field offset (16-byte units) of slice s in a stage: the
// low half-record box holds slices 0-3 at 32-byte steps, the high box 4-7
__host__ __device__ constexpr uint64_t oz_slice_off(int s) { return (uint64_t)((s >> 2) * (kOzBox >> 4) + 2 * (s & 3)); }

// the highest d-group an off-diagonal Gram tile accumulates: every d = s + s'
// <= 6 for seven-slice data, d <= 3 (pass 1 only) for four-slice data.
// Diagonal tiles keep every d-group up to 6, so each G[t][t] carries the
// dropped groups (whose terms q_s q_s' add coherently there, all positive for
// s = s'); off the diagonal the dropped terms are sums of uncorrelated low
// digits, relative ~1/sqrt(V): for fp32 data on the BASELINE recipe (V = 30k)
// ~1e-8 of |G| normwise, 3e-9 of A^T A = S G S^T / 4 and ~2e-9 of W^T W - I
// (tools/slice_drop_probe.py), against fp32's 1e-4 parity tolerance and
// criterion 4's 1e-8; it saves pass 2 on 97% of the tiles (cfg 4: 99 -> 64
// ms).  Subjects of fewer than kOzDropMinBlocks * 32 voxels keep every pair
// (their Grams are cheap, and W^T W - I would reach ~5e-9 at V = 2600).
// Seven-slice data keeps d = 6 off the diagonal too: dropping it saved 2%
// (pass 2 is bound by its operand traffic, not the MMAs) for 100x the error.
__host__ __device__ constexpr int oz_dtop_off(int nsl) { return nsl > 4 ? 6 : 3; }
constexpr int kOzDropMinBlocks = 512;

// the MMAs of one 32-voxel block in pass P: d-groups 0-3 (P = 0) or 4-DTOP
// (P = 1), pairs s + s' = d with s, s' < NSL, fully unrolled; `keep` = 0
// starts the accumulators (first block of a chunk)
template <int NSL, int P, int DTOP = kOzSlices - 1>
__device__ __forceinline__ void oz_issue_pass(uint32_t tmem, uint64_t da0, uint64_t db0, uint32_t idesc,
                                              uint32_t keep) {
  constexpr int dlo = P ? 4 : 0, dhi = P ? DTOP : 3;
#pragma unroll
  for (int d = dlo; d <= dhi; ++d) {
    const uint32_t acc = tmem + 128u * (uint32_t)(d - dlo);
    const int s0 = d - (NSL - 1) > 0 ? d - (NSL - 1) : 0, s1 = d < NSL - 1 ? d : NSL - 1;
#pragma unroll
    for (int s = s0; s <= s1; ++s)
      mma_s8(acc, da0 + oz_slice_off(s), db0 + oz_slice_off(d - s), idesc, s == s0 ? keep : 1u);
  }
}

// N of a Gram tile's MMAs: the 16-column multiple covering the columns
// below o.nmma (T), at most 128 -- the last column block of T = 1000 (ldx
// 1024) needs 112, so its eight tiles issue 12.5% fewer MACs
__device__ __forceinline__ int oz_tile_n(const OzGramOut& o, int n0) {
  const int64_t lim = o.nmma > 0 ? o.nmma : o.nout;
  const int64_t c = lim - n0;
  return c >= 128 ? 128 : (c <= 16 ? 16 : (int)((c + 15) & ~15));
}

template <int NSL>
__global__ void __launch_bounds__(kOzThreads, 1) k_oz_gram(const __grid_constant__ CUtensorMap tmq,
                                                           const OzGramOut o, const OzItem* __restrict__ items) {
  constexpr int nsl = NSL;  // compile time: the MMA issue loops unroll
  // d-groups 0..3 fill the 512 TMEM columns; pass 2 accumulates d = 4..6 on
  // diagonal tiles, d = 4..5 off the diagonal (oz_dtop_off); four-slice data
  // off the diagonal needs no pass 2
  extern __shared__ __align__(1024) unsigned char oz_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ OzBars bars;
  __shared__ uint32_t tmem_base;
  const OzItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvb = it.nvb;
  const bool diag = it.m0 == it.n0;
  const bool all_d = diag || nvb < kOzDropMinBlocks;  // every d-group (oz_dtop_off)
  const int nchunks = (nvb + kOzChunkBlocks - 1) / kOzChunkBlocks;
  const int kPasses = (oz_dtop_off(nsl) < 4 && !all_d) ? 1 : 2;

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < kOzStages; ++s) {
        mbar_init(&bars.full[s], 1);
        mbar_init(&bars.empty[s], 1);
      }
      mbar_init(&bars.accfull, 1);
      mbar_init(&bars.accfree, kOzThreads - 64);
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
  } else if (warp == 1) {
    tmem_alloc(&tmem_base, 512);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int k = 0;
      for (int c = 0; c < nchunks; ++c) {
        const int b0 = c * kOzChunkBlocks, b1 = min(nvb, b0 + kOzChunkBlocks);
        for (int pass = 0; pass < kPasses; ++pass) {
          // slices 4..6 (the records' high halves) only for pass 2 of seven-slice
          // data; a low-half-only pass packs two 32-voxel blocks per stage
          const bool hi = pass && nsl > 4;
          const int step = hi ? 1 : 2;
          for (int vb = b0; vb < b1; vb += step, ++k) {
            const int slot = k % kOzStages;
            if (k >= kOzStages) mbar_wait(&bars.empty[slot], ((k / kOzStages) - 1) & 1);
            const int nj = min(step, b1 - vb);
            const int nbox = (hi ? 2 : nj) * (diag ? 1 : 2);
            mbar_expect_tx(&bars.full[slot], (uint32_t)(nbox * kOzBox));
            unsigned char* st = smem + slot * kOzStageBytes;
            const int x = (it.vb0 + vb) * oz_record_bytes(nsl);
            if (hi) {  // [A lo][A hi][B lo][B hi]
              tma_load_3d(st, &tmq, x, it.m0, it.subj, &bars.full[slot]);
              tma_load_3d(st + kOzBox, &tmq, x + 128, it.m0, it.subj, &bars.full[slot]);
              if (!diag) {
                tma_load_3d(st + 2 * kOzBox, &tmq, x, it.n0, it.subj, &bars.full[slot]);
                tma_load_3d(st + 3 * kOzBox, &tmq, x + 128, it.n0, it.subj, &bars.full[slot]);
              }
            } else {   // [A lo vb][A lo vb + 1][B lo vb][B lo vb + 1]
              for (int j = 0; j < nj; ++j) {
                const int xj = (it.vb0 + vb + j) * oz_record_bytes(nsl);
                tma_load_3d(st + j * kOzBox, &tmq, xj, it.m0, it.subj, &bars.full[slot]);
                if (!diag) tma_load_3d(st + (2 + j) * kOzBox, &tmq, xj, it.n0, it.subj, &bars.full[slot]);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = idesc_s8(128, oz_tile_n(o, it.n0));
      int k = 0, npass = 0;
      for (int c = 0; c < nchunks; ++c) {
        const int b0 = c * kOzChunkBlocks, b1 = min(nvb, b0 + kOzChunkBlocks);
        for (int pass = 0; pass < kPasses; ++pass, ++npass) {
          // the epilogue must have drained the previous pass's accumulators
          if (npass > 0) mbar_wait(&bars.accfree, (npass - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const bool hi = pass && nsl > 4;
          const int step = hi ? 1 : 2;
          for (int vb = b0; vb < b1; vb += step, ++k) {
            const int slot = k % kOzStages;
            mbar_wait(&bars.full[slot], (k / kOzStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t sa = smem_u32(smem + slot * kOzStageBytes);
            const uint32_t sb = diag ? sa : sa + 2 * kOzBox;
            // one descriptor per operand; slices are fixed offsets added to
            // its address field, so each MMA costs two 64-bit adds to issue
            const uint64_t da0 = umma_desc_sw128(sa), db0 = umma_desc_sw128(sb);
            const uint32_t keep = vb == b0 ? 0u : 1u;
            if (hi) {
              if (all_d)
                oz_issue_pass<nsl, 1>(tmem, da0, db0, idesc, keep);
              else
                oz_issue_pass<nsl, 1, oz_dtop_off(nsl)>(tmem, da0, db0, idesc, keep);
            } else {
              // the stage's second block sits one box after the first (A and B alike)
              const uint64_t box = (uint64_t)(kOzBox >> 4);
              const int nj = min(step, b1 - vb);
              if (pass == 0) {
                oz_issue_pass<nsl, 0>(tmem, da0, db0, idesc, keep);
                if (nj > 1) oz_issue_pass<nsl, 0>(tmem, da0 + box, db0 + box, idesc, 1u);
              } else {
                oz_issue_pass<nsl, 1>(tmem, da0, db0, idesc, keep);
                if (nj > 1) oz_issue_pass<nsl, 1>(tmem, da0 + box, db0 + box, idesc, 1u);
              }
            }
            mma_commit(&bars.empty[slot]);
          }
          mma_commit(&bars.accfull);
        }
      }
    }
  } else {
    // ---------------- epilogue: warps 2-9, TMEM lanes 32 (warp % 4), 64-column halves ----------------
    const int quarter = warp & 3;
    const int cbase = ((warp - 2) >> 2) * 64;
    const int r = quarter * 32 + lane;
    const int64_t ta = it.m0 + r;
    const bool rin = ta < o.nout;
    const int32_t* ex = o.expo + (int64_t)it.subj * o.ldexp;
    const int ea = ta < o.nexp ? ex[ta] : 0;
    double* grow = o.g + (int64_t)it.slot * o.gsub + ta * o.ldg + it.n0;
    const int tn = oz_tile_n(o, it.n0);
    int npass = 0;
    for (int c = 0; c < nchunks; ++c) {
      for (int pass = 0; pass < kPasses; ++pass, ++npass) {
        mbar_wait(&bars.accfull, npass & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        // d-groups dlo..dtop were accumulated; the sum is weighted as dlo..dhi
        const int dlo = pass ? 4 : 0, dhi = pass ? kOzSlices - 1 : 3;
        const int dtop = pass ? (all_d ? kOzSlices - 1 : oz_dtop_off(nsl)) : 3;
        for (int c0 = cbase; c0 < cbase + 64; c0 += 16) {
          // pass 2 adds to pass 1's values: their loads go out first
          double prev[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            prev[j] = (npass > 0 && rin && it.n0 + c0 + j < o.nout) ? grow[c0 + j] : 0.0;
          // the (up to four) d-groups of these 16 columns in flight, one wait
          uint32_t raw[4][16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (dlo + q <= dtop)
              tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + 128u * (uint32_t)q + c0, raw[q]);
            else
#pragma unroll
              for (int j = 0; j < 16; ++j) raw[q][j] = 0u;
          }
          tmem_wait_ld();
          // the pass's d-groups as one exact int64 (|raw| < 2^31): pass 1
          // H = sum_{d<4} raw_d 2^{7(3-d)} (x 2^-33), pass 2 L = sum_{d>=4}
          // raw_d 2^{7(6-d)} (x 2^-54) -- one conversion and one rounding
          double val[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            long long h = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (dlo + q <= dhi) h = h * 128 + (long long)(int32_t)raw[q][j];
            val[j] = (double)h * (pass ? 0x1p-54 : 0x1p-33);
          }
          if (rin) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int64_t tb = it.n0 + c0 + j;
              if (tb < o.nout) {
                // columns past the trimmed N are the zeros of X-hat's padded TRs
                const double g = c0 + j < tn ? val[j] * pow2(ea + (tb < o.nexp ? ex[tb] : 0)) : 0.0;
                grow[c0 + j] = (npass == 0) ? g : prev[j] + g;
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(&bars.accfree);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) tmem_free(tmem, 512);
}

// ---------------------------------------------------------------------------
// gram tiles on CTA pairs: tcgen05.mma.cta_group::2, M = 256 (two 128-row
// blocks of the Gram, one per CTA) x N = 128.  Each CTA stages its own 128 A
// rows and half of the B rows (64), so a CTA's shared-memory operand reads per
// MMA drop from 8 KB to 6 KB and its TMA writes by a quarter -- the
// single-CTA kernel is bound by the tensor core's shared-memory port (ncu:
// sm__mem_tensor_cycles_active 85%).  Both producers signal the leader's full
// barrier (cta_group::2 TMA), the leader issues every MMA and multicasts its
// commits to both CTAs' empty / accumulator barriers, and every epilogue warp
// of the pair arrives on the leader's accumulator-free barrier.  Pairs cover
// the upper 128-tiles of a column block two row blocks at a time; a tile below
// the diagonal is computed and discarded (mirror_gram fills the lower half).
// ---------------------------------------------------------------------------
constexpr int kOz2Stages = 4;
constexpr int kOzBoxB = 8192;  // 64 rows x 128 bytes
constexpr int kOz2StageBytes = 2 * kOzBox + 2 * kOzBoxB;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}

__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
      : "memory");
}

__device__ __forceinline__ void mma_s8_pair(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3));
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// slice s of an operand staged as [lo box][hi box] of `box` bytes each
__host__ __device__ constexpr uint64_t oz_slice_off_box(int s, int box) {
  return (uint64_t)((s >> 2) * (box >> 4) + 2 * (s & 3));
}

template <int NSL, int P, int DTOP = kOzSlices - 1>
__device__ __forceinline__ void oz_issue_pass_pair(uint32_t tmem, uint64_t da0, uint64_t db0, uint32_t idesc,
                                                   uint32_t keep) {
  constexpr int dlo = P ? 4 : 0, dhi = P ? DTOP : 3;
#pragma unroll
  for (int d = dlo; d <= dhi; ++d) {
    const uint32_t acc = tmem + 128u * (uint32_t)(d - dlo);
    const int s0 = d - (NSL - 1) > 0 ? d - (NSL - 1) : 0, s1 = d < NSL - 1 ? d : NSL - 1;
#pragma unroll
    for (int s = s0; s <= s1; ++s)
      mma_s8_pair(acc, da0 + oz_slice_off_box(s, kOzBox), db0 + oz_slice_off_box(d - s, kOzBoxB), idesc,
                  s == s0 ? keep : 1u);
  }
}

template <int NSL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kOzThreads, 1)
    k_oz_gram2(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmqb, const OzGramOut o,
               const OzItem* __restrict__ items) {
  constexpr int nsl = NSL;
  extern __shared__ __align__(1024) unsigned char oz_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kOz2Stages], empty[kOz2Stages], accfull, accfree;
  __shared__ uint32_t tmem_base;
  const uint32_t rank = cluster_rank();
  const OzItem it = items[blockIdx.x >> 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvb = it.nvb;
  const int nchunks = (nvb + kOzChunkBlocks - 1) / kOzChunkBlocks;
  // B's N columns split between the pair at N / 2 (N = 128, or trimmed to T
  // on the last column block): CTA r stages rows n0 + r N / 2 ..
  const int arow = it.m0 + 128 * (int)rank, brow = it.n0 + (oz_tile_n(o, it.n0) / 2) * (int)rank;
  // the d-groups are k_oz_gram's per tile: the pair accumulates the union
  // (every group when either tile is diagonal) and each epilogue takes its own
  const bool small = it.nvb < kOzDropMinBlocks;
  const bool mydiag = arow == it.n0 || small, anydiag = it.m0 == it.n0 || it.m0 + 128 == it.n0 || small;
  const int kPasses = (oz_dtop_off(nsl) < 4 && !anydiag) ? 1 : 2;

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < kOz2Stages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(&accfull, 1);
      mbar_init(&accfree, 2 * (kOzThreads - 64) / 32);  // every epilogue warp of the pair
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
  } else if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ---------------- TMA producers (both CTAs), the leader's full barriers ----------------
    if (lane == 0) {
      int k = 0;
      for (int c = 0; c < nchunks; ++c) {
        const int b0 = c * kOzChunkBlocks, b1 = min(nvb, b0 + kOzChunkBlocks);
        for (int pass = 0; pass < kPasses; ++pass) {
          const bool hi = pass && nsl > 4;
          const int step = hi ? 1 : 2;
          for (int vb = b0; vb < b1; vb += step, ++k) {
            const int slot = k % kOz2Stages;
            if (k >= kOz2Stages) mbar_wait(&empty[slot], ((k / kOz2Stages) - 1) & 1);
            const int nj = min(step, b1 - vb);
            if (rank == 0)  // both CTAs' bytes land on the leader's barrier
              mbar_expect_tx(&full[slot], (uint32_t)(2 * (hi ? 2 * (kOzBox + kOzBoxB) : nj * (kOzBox + kOzBoxB))));
            const uint32_t fb = leader_addr(&full[slot]);
            unsigned char* st = smem + slot * kOz2StageBytes;
            unsigned char* sb = st + 2 * kOzBox;
            if (hi) {  // [A lo][A hi][B lo][B hi]
              const int x = (it.vb0 + vb) * oz_record_bytes(nsl);
              tma_load_3d_pair(st, &tmq, x, arow, it.subj, fb);
              tma_load_3d_pair(st + kOzBox, &tmq, x + 128, arow, it.subj, fb);
              tma_load_3d_pair(sb, &tmqb, x, brow, it.subj, fb);
              tma_load_3d_pair(sb + kOzBoxB, &tmqb, x + 128, brow, it.subj, fb);
            } else {   // [A lo vb][A lo vb + 1][B lo vb][B lo vb + 1]
              for (int j = 0; j < nj; ++j) {
                const int xj = (it.vb0 + vb + j) * oz_record_bytes(nsl);
                tma_load_3d_pair(st + j * kOzBox, &tmq, xj, arow, it.subj, fb);
                tma_load_3d_pair(sb + j * kOzBoxB, &tmqb, xj, brow, it.subj, fb);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only) ----------------
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = idesc_s8(256, oz_tile_n(o, it.n0));
      int k = 0, npass = 0;
      for (int c = 0; c < nchunks; ++c) {
        const int b0 = c * kOzChunkBlocks, b1 = min(nvb, b0 + kOzChunkBlocks);
        for (int pass = 0; pass < kPasses; ++pass, ++npass) {
          if (npass > 0) mbar_wait(&accfree, (npass - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const bool hi = pass && nsl > 4;
          const int step = hi ? 1 : 2;
          for (int vb = b0; vb < b1; vb += step, ++k) {
            const int slot = k % kOz2Stages;
            mbar_wait(&full[slot], (k / kOz2Stages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t sa = smem_u32(smem + slot * kOz2StageBytes);
            const uint64_t da0 = umma_desc_sw128(sa), db0 = umma_desc_sw128(sa + 2 * kOzBox);
            const uint32_t keep = vb == b0 ? 0u : 1u;
            if (hi) {
              if (anydiag)
                oz_issue_pass_pair<nsl, 1>(tmem, da0, db0, idesc, keep);
              else
                oz_issue_pass_pair<nsl, 1, oz_dtop_off(nsl)>(tmem, da0, db0, idesc, keep);
            } else {
              const uint64_t boxa = (uint64_t)(kOzBox >> 4), boxb = (uint64_t)(kOzBoxB >> 4);
              const int nj = min(step, b1 - vb);
              if (pass == 0) {
                oz_issue_pass_pair<nsl, 0>(tmem, da0, db0, idesc, keep);
                if (nj > 1) oz_issue_pass_pair<nsl, 0>(tmem, da0 + boxa, db0 + boxb, idesc, 1u);
              } else {
                oz_issue_pass_pair<nsl, 1>(tmem, da0, db0, idesc, keep);
                if (nj > 1) oz_issue_pass_pair<nsl, 1>(tmem, da0 + boxa, db0 + boxb, idesc, 1u);
              }
            }
            mma_commit_pair(&empty[slot]);
          }
          mma_commit_pair(&accfull);
        }
      }
    }
  } else {
    // ---------------- epilogue: warps 2-9 of each CTA, its own 128 rows ----------------
    const int quarter = warp & 3;
    const int cbase = ((warp - 2) >> 2) * 64;
    const int r = quarter * 32 + lane;
    const int64_t ta = arow + r;
    const bool below = (arow / 128) > (it.n0 / 128);  // a tile below the diagonal: discarded
    const bool rin = ta < o.nout && !below;
    const int32_t* ex = o.expo + (int64_t)it.subj * o.ldexp;
    const int ea = ta < o.nexp ? ex[ta] : 0;
    double* grow = o.g + (int64_t)it.slot * o.gsub + ta * o.ldg + it.n0;
    const int tn = oz_tile_n(o, it.n0);
    const uint32_t freebar = leader_addr(&accfree);
    int npass = 0;
    for (int c = 0; c < nchunks; ++c) {
      for (int pass = 0; pass < kPasses; ++pass, ++npass) {
        mbar_wait(&accfull, npass & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int dlo = pass ? 4 : 0, dhi = pass ? kOzSlices - 1 : 3;
        const int dtop = pass ? (mydiag ? kOzSlices - 1 : oz_dtop_off(nsl)) : 3;
        if (!below && dlo <= dtop) {
          for (int c0 = cbase; c0 < cbase + 64; c0 += 16) {
            double prev[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              prev[j] = (npass > 0 && rin && it.n0 + c0 + j < o.nout) ? grow[c0 + j] : 0.0;
            uint32_t raw[4][16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (dlo + q <= dtop)
                tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + 128u * (uint32_t)q + c0, raw[q]);
              else
#pragma unroll
                for (int j = 0; j < 16; ++j) raw[q][j] = 0u;
            }
            tmem_wait_ld();
            double val[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              long long h = 0;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (dlo + q <= dhi) h = h * 128 + (long long)(int32_t)raw[q][j];
              val[j] = (double)h * (pass ? 0x1p-54 : 0x1p-33);
            }
            if (rin) {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const int64_t tb = it.n0 + c0 + j;
                if (tb < o.nout) {
                  const double g = c0 + j < tn ? val[j] * pow2(ea + (tb < o.nexp ? ex[tb] : 0)) : 0.0;
                  grow[c0 + j] = (npass == 0) ? g : prev[j] + g;
                }
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(freebar);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---------------------------------------------------------------------------
// B_i = G_i^T Xhat_i on the int8 tensor cores (the E-step term of the initial
// mapping, srm.py:101-118: W_0 = G M_0, so W_0^T Xhat = M_0^T (G^T Xhat)).
// The same machinery as k_oz_gram with two record tensors: A = the seven
// slices of the N(0,1) draw G (records [k][32-voxel block], the draw's column
// scales), B = Xhat's slices (seven or four) -- one M = 128 feature tile by
// N = 128 TRs per CTA, contracted over the subject's voxels.  Pairs
// (s, s') with s + s' <= 6 (all of them for four-slice Xhat); the result goes
// to the subject's reduced record (bred[i][k][t], row stride ldo) for k < kp.
// ---------------------------------------------------------------------------
template <int NSA, int NSB, int P>
__device__ __forceinline__ void oz_issue_pass_ab(uint32_t tmem, uint64_t da0, uint64_t db0, uint32_t idesc,
                                                 uint32_t keep) {
  constexpr int dlo = P ? 4 : 0, dhi = P ? kOzSlices - 1 : 3;
#pragma unroll
  for (int d = dlo; d <= dhi; ++d) {
    const uint32_t acc = tmem + 128u * (uint32_t)(d - dlo);
    const int s0 = d - (NSB - 1) > 0 ? d - (NSB - 1) : 0, s1 = d < NSA - 1 ? d : NSA - 1;
#pragma unroll
    for (int s = s0; s <= s1; ++s)
      mma_s8(acc, da0 + oz_slice_off(s), db0 + oz_slice_off(d - s), idesc, s == s0 ? keep : 1u);
  }
}

struct OzTnArgs {
  const int32_t* aexp;  // [n_local][K] column exponents of G
  const int32_t* bexp;  // [n_local][ldx] column exponents of Xhat
  double* out;          // bred
  int64_t ldx, kp, ldo, K;
};

template <int NSB>
__global__ void __launch_bounds__(kOzThreads, 1) k_oz_tn(const __grid_constant__ CUtensorMap tma,
                                                         const __grid_constant__ CUtensorMap tmb, OzTnArgs g,
                                                         const OzItem* __restrict__ items) {
  constexpr int NSA = kOzSlices;
  constexpr int recb = NSB <= 4 ? 128 : 256;
  // four-slice (fp32) Xhat: the pairs s + s' <= 3 only, one pass.  The dropped
  // pairs are products of independent low digits of G and Xhat: ~1e-7 of
  // |G^T Xhat| normwise on the BASELINE recipe, where the 2^-27 truncation of
  // Xhat itself already costs ~1e-8 (fp32 parity tolerance: 1e-4)
  constexpr int kPasses = NSB <= 4 ? 1 : 2;
  extern __shared__ __align__(1024) unsigned char oz_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ OzBars bars;
  __shared__ uint32_t tmem_base;
  const OzItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvb = it.nvb;
  const int nchunks = (nvb + kOzChunkBlocks - 1) / kOzChunkBlocks;

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < kOzStages; ++s) {
        mbar_init(&bars.full[s], 1);
        mbar_init(&bars.empty[s], 1);
      }
      mbar_init(&bars.accfull, 1);
      mbar_init(&bars.accfree, kOzThreads - 64);
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
  } else if (warp == 1) {
    tmem_alloc(&tmem_base, 512);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int k = 0;
      for (int c = 0; c < nchunks; ++c) {
        const int b0 = c * kOzChunkBlocks, b1 = min(nvb, b0 + kOzChunkBlocks);
        for (int pass = 0; pass < kPasses; ++pass) {
          // pass 1 reads G's high halves (slices 4-6) and, for seven-slice
          // Xhat, its high halves too; the low-half pass packs two blocks a stage
          const bool hi = pass != 0;
          const int step = hi ? 1 : 2;
          for (int vb = b0; vb < b1; vb += step, ++k) {
            const int slot = k % kOzStages;
            if (k >= kOzStages) mbar_wait(&bars.empty[slot], ((k / kOzStages) - 1) & 1);
            const int nj = min(step, b1 - vb);
            const int nbox = hi ? (NSB > 4 ? 4 : 3) : 2 * nj;
            mbar_expect_tx(&bars.full[slot], (uint32_t)(nbox * kOzBox));
            unsigned char* st = smem + slot * kOzStageBytes;
            if (hi) {  // [A lo][A hi][B lo][B hi]
              tma_load_3d(st, &tma, vb * 256, 0, it.subj, &bars.full[slot]);
              tma_load_3d(st + kOzBox, &tma, vb * 256 + 128, 0, it.subj, &bars.full[slot]);
              tma_load_3d(st + 2 * kOzBox, &tmb, vb * recb, it.n0, it.subj, &bars.full[slot]);
              if (NSB > 4) tma_load_3d(st + 3 * kOzBox, &tmb, vb * recb + 128, it.n0, it.subj, &bars.full[slot]);
            } else {   // [A lo vb][A lo vb + 1][B lo vb][B lo vb + 1]
              for (int j = 0; j < nj; ++j) {
                tma_load_3d(st + j * kOzBox, &tma, (vb + j) * 256, 0, it.subj, &bars.full[slot]);
                tma_load_3d(st + (2 + j) * kOzBox, &tmb, (vb + j) * recb, it.n0, it.subj, &bars.full[slot]);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_s8(128, 128);
      int k = 0, npass = 0;
      for (int c = 0; c < nchunks; ++c) {
        const int b0 = c * kOzChunkBlocks, b1 = min(nvb, b0 + kOzChunkBlocks);
        for (int pass = 0; pass < kPasses; ++pass, ++npass) {
          if (npass > 0) mbar_wait(&bars.accfree, (npass - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const bool hi = pass != 0;
          const int step = hi ? 1 : 2;
          for (int vb = b0; vb < b1; vb += step, ++k) {
            const int slot = k % kOzStages;
            mbar_wait(&bars.full[slot], (k / kOzStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t sa = smem_u32(smem + slot * kOzStageBytes);
            const uint64_t da0 = umma_desc_sw128(sa), db0 = umma_desc_sw128(sa + 2 * kOzBox);
            const uint32_t keep = vb == b0 ? 0u : 1u;
            if (hi) {
              oz_issue_pass_ab<NSA, NSB, 1>(tmem, da0, db0, idesc, keep);
            } else {
              const uint64_t box = (uint64_t)(kOzBox >> 4);
              oz_issue_pass_ab<NSA, NSB, 0>(tmem, da0, db0, idesc, keep);
              if (min(step, b1 - vb) > 1) oz_issue_pass_ab<NSA, NSB, 0>(tmem, da0 + box, db0 + box, idesc, 1u);
            }
            mma_commit(&bars.empty[slot]);
          }
          mma_commit(&bars.accfull);
        }
      }
    }
  } else {
    // ---------------- epilogue: warps 2-9, TMEM lanes 32 (warp % 4), 64-column halves ----------------
    const int quarter = warp & 3;
    const int cbase = ((warp - 2) >> 2) * 64;
    const int r = quarter * 32 + lane;  // feature k
    const bool rin = r < g.kp;
    const int ea = r < g.K ? g.aexp[(int64_t)it.subj * g.K + r] : 0;
    const int32_t* ex = g.bexp + (int64_t)it.subj * g.ldx;
    double* orow = g.out + (int64_t)it.subj * g.kp * g.ldo + (int64_t)r * g.ldo + it.n0;
    int npass = 0;
    for (int c = 0; c < nchunks; ++c) {
      for (int pass = 0; pass < kPasses; ++pass, ++npass) {
        mbar_wait(&bars.accfull, npass & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int dlo = pass ? 4 : 0, dhi = pass ? kOzSlices - 1 : 3;
        for (int c0 = cbase; c0 < cbase + 64; c0 += 16) {
          double prev[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) prev[j] = (npass > 0 && rin && it.n0 + c0 + j < g.ldx) ? orow[c0 + j] : 0.0;
          uint32_t raw[4][16];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (dlo + q <= dhi) tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + 128u * (uint32_t)q + c0, raw[q]);
          tmem_wait_ld();
          double val[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            long long h = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (dlo + q <= dhi) h = h * 128 + (long long)(int32_t)raw[q][j];
            val[j] = (double)h * (pass ? 0x1p-54 : 0x1p-33);
          }
          if (rin) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int64_t tb = it.n0 + c0 + j;
              if (tb < g.ldx) {
                const double v = val[j] * pow2(ea + ex[tb]);
                orow[c0 + j] = (npass == 0) ? v : prev[j] + v;
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(&bars.accfree);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) tmem_free(tmem, 512);
}

// The same B_i = G_i^T Xhat_i for kp <= 64, transposed: M = 128 TRs (the
// X-hat records) x N = 64 features (the draw's records), so a K = 50 tile
// wastes 14 of 64 columns instead of 78 of 128 rows, and all seven 64-column
// d-groups fit the 512 TMEM columns at once -- one pass over the slices, the
// exact int64 combination of both d-group halves in one epilogue.
template <int NSX>
__global__ void __launch_bounds__(kOzThreads, 1) k_oz_nt(const __grid_constant__ CUtensorMap tmx,
                                                         const __grid_constant__ CUtensorMap tmg, OzTnArgs g,
                                                         const OzItem* __restrict__ items) {
  constexpr int NSG = kOzSlices;
  constexpr int recx = NSX <= 4 ? 128 : 256;
  constexpr int kDTop = NSX <= 4 ? 3 : kOzSlices - 1;  // k_oz_tn's d-groups (bit-identical results)
  constexpr int kBoxG = 8192;                          // 64 rows x 128 B
  constexpr int kStage = (NSX > 4 ? 2 : 1) * kOzBox + 2 * kBoxG;
  constexpr int kSt = 4;
  extern __shared__ __align__(1024) unsigned char oz_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kSt], empty[kSt], accfull, accfree;
  __shared__ uint32_t tmem_base;
  const OzItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvb = it.nvb;
  const int nchunks = (nvb + kOzChunkBlocks - 1) / kOzChunkBlocks;

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < kSt; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(&accfull, 1);
      mbar_init(&accfree, kOzThreads - 64);
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
  } else if (warp == 1) {
    tmem_alloc(&tmem_base, 512);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer: [X lo][X hi][G lo][G hi] per 32-voxel block
      int k = 0;
      for (int c = 0; c < nchunks; ++c) {
        const int b0 = c * kOzChunkBlocks, b1 = min(nvb, b0 + kOzChunkBlocks);
        for (int vb = b0; vb < b1; ++vb, ++k) {
          const int slot = k % kSt;
          if (k >= kSt) mbar_wait(&empty[slot], ((k / kSt) - 1) & 1);
          mbar_expect_tx(&full[slot], (uint32_t)(kDTop >= 4 ? kStage : kStage - kBoxG));
          unsigned char* st = smem + slot * kStage;
          tma_load_3d(st, &tmx, vb * recx, it.n0, it.subj, &full[slot]);
          if (NSX > 4) tma_load_3d(st + kOzBox, &tmx, vb * recx + 128, it.n0, it.subj, &full[slot]);
          // the draw's slots of this voxel block as [slot][64 features][32 B] (SWIZZLE_32B):
          // slots j, j + 1 form one 128-row K-major operand
          unsigned char* sg = st + (NSX > 4 ? 2 : 1) * kOzBox;
          tma_load_4d(sg, &tmg, 0, 0, vb * 8, it.subj, &full[slot]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer: seven 64-column d-groups, one pass
      // N = 128: B is the slot pair (s2, s2 + 1) of the draw, 64 features each, so one MMA
      // feeds d-groups sx + s2 and sx + s2 + 1 (adjacent accumulators) -- 16 MMAs per voxel
      // block instead of 28 at N = 64, which cost the same tensor-pipe time each
      // (tools/i8_peak.cu); the same integer sums per d-group, so the result is unchanged.
      // A partial group past kDTop is written and never read.
      constexpr uint32_t idesc = idesc_s8(128, 128);
      int k = 0;
      for (int c = 0; c < nchunks; ++c) {
        if (c > 0) mbar_wait(&accfree, (c - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int b0 = c * kOzChunkBlocks, b1 = min(nvb, b0 + kOzChunkBlocks);
        for (int vb = b0; vb < b1; ++vb, ++k) {
          const int slot = k % kSt;
          mbar_wait(&full[slot], (k / kSt) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(smem + slot * kStage);
          const uint64_t da0 = umma_desc_sw128(sa);
          const uint64_t db0 = umma_desc_sw32_mn(sa + (NSX > 4 ? 2 : 1) * kOzBox, 16, 256);
          const uint32_t keep = vb == b0 ? 0u : 1u;
          // sx = 0 first: its pairs touch every d-group read, so they alone start a chunk's sums
#pragma unroll
          for (int sx = 0; sx < NSX; ++sx)
#pragma unroll
            for (int s2 = 0; sx + s2 <= kDTop; s2 += 2)
              mma_s8(tmem + 64u * (uint32_t)(sx + s2), da0 + oz_slice_off_box(sx, kOzBox),
                     db0 + (uint64_t)(s2 * (2048 >> 4)), idesc, sx == 0 ? keep : 1u);
          mma_commit(&empty[slot]);
        }
        mma_commit(&accfull);
      }
    }
  } else {
    // ---------------- epilogue: warps 2-9; TMEM lane = TR, 32-feature halves ----------------
    const int quarter = warp & 3;
    const int kbase = ((warp - 2) >> 2) * 32;
    const int r = quarter * 32 + lane;
    const int64_t t = it.n0 + r;
    const bool tin = t < g.ldx;
    const int et = tin ? g.bexp[(int64_t)it.subj * g.ldx + t] : 0;
    const int32_t* ek = g.aexp + (int64_t)it.subj * g.K;
    double* ocol = g.out + (int64_t)it.subj * g.kp * g.ldo + t;  // out[k][t] = ocol[k * ldo]
    for (int c = 0; c < nchunks; ++c) {
      mbar_wait(&accfull, c & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int k0 = kbase; k0 < kbase + 32; k0 += 16) {
        uint32_t raw[kOzSlices][16];
#pragma unroll
        for (int d = 0; d < kOzSlices; ++d) {
          if (d <= kDTop)
            tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + 64u * (uint32_t)d + k0, raw[d]);
          else
#pragma unroll
            for (int j = 0; j < 16; ++j) raw[d][j] = 0u;
        }
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int kk = k0 + j;
          if (!tin || kk >= g.kp) continue;
          long long h = 0, l = 0;
#pragma unroll
          for (int d = 0; d < 4; ++d) h = h * 128 + (long long)(int32_t)raw[d][j];
#pragma unroll
          for (int d = 4; d < kOzSlices; ++d) l = l * 128 + (long long)(int32_t)raw[d][j];
          // the two-pass kernel's arithmetic: (double) H 2^-33, then + (double) L 2^-54
          const double sc = pow2(et + (kk < g.K ? ek[kk] : 0));
          const double v0 = (double)h * 0x1p-33 * sc;
          const double v1 = (double)l * 0x1p-54 * sc;
          double* o = ocol + (int64_t)kk * g.ldo;
          *o = (c == 0) ? v0 + v1 : (*o + v0) + v1;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&accfree);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) tmem_free(tmem, 512);
}

// column maxima |a[:, c]| of each subject's rows (c < ncols), as IEEE bits: one
// CTA per 256 rows, eight row groups reduced in shared memory, one atomic per
// column per CTA
__global__ void __launch_bounds__(256) k_oz_colmax(DevPlan p, const double* __restrict__ a, int64_t lda, int ncols,
                                                   unsigned long long* __restrict__ cmax) {
  __shared__ double red[8][33];
  const int i = p.sub0 + blockIdx.y;
  const int64_t* sj = p.subj + (int64_t)i * kSubjCols;
  const int64_t row0 = sj[SC_ROW_OFF], V = sj[SC_V];
  const int lane = threadIdx.x & 31, rsub = threadIdx.x >> 5;
  const int64_t v1 = min(V, (int64_t)(blockIdx.x + 1) * 256);
  for (int c0 = 0; c0 < ncols; c0 += 32) {
    const int col = c0 + lane;
    double m = 0.0;
    if (col < ncols)
      for (int64_t v = (int64_t)blockIdx.x * 256 + rsub; v < v1; v += 8) m = fmax(m, fabs(a[(row0 + v) * lda + col]));
    red[rsub][lane] = m;
    __syncthreads();
    if (rsub == 0) {
      for (int r = 1; r < 8; ++r) m = fmax(m, red[r][lane]);
      if (col < ncols && m > 0.0)
        atomicMax(&cmax[(int64_t)i * ncols + col], (unsigned long long)__double_as_longlong(m));
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// row slicing: one warp per row of a row-major fp64 matrix M (rows x ldm,
// columns [0, ncols), ncols % 32 == 0); the row's power-of-two scale 2^e >=
// max |M[r][:]| goes to expo[r] and its slices to the 256-byte records
// q[r][b] (b = 32-column block), the same record layout as oz_split, or --
// tile_rows > 0, the G_i of the int8 B = S G / 2 (tile_rows = rows per G_i) --
// tiled: [subject][128-row block][32-column block][record half][128 rows][128 B],
// so each k-block of an M = 128 tile is one contiguous 32 KB read.
// Matrices: the fp64 Gram G_i (rows = TRs, once) and S (rows = features,
// every iteration) of the int8 B = S G / 2.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_oz_slice_rows(const double* __restrict__ M, int64_t ldm, int64_t rows,
                                                       int64_t ncols, int8_t* __restrict__ q, int64_t lq,
                                                       int32_t* __restrict__ expo, int64_t tile_rows) {
  __shared__ __align__(16) uint8_t rec[8][kOzRecord];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + warp;
  if (r >= rows) return;
  const double* row = M + r * ldm;
  double m = 0.0;
  for (int64_t c0 = 0; c0 < ncols; c0 += 256) {  // eight loads in flight per lane
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t c = c0 + lane + 32 * u;
      v[u] = c < ncols ? fabs(row[c]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) m = fmax(m, v[u]);
  }
  m = warp_max(m);
  const int e = (m > 0.0) ? frexp_exp(m) : 0;
  if (lane == 0) expo[r] = e;
  const double scale = __longlong_as_double((long long)(1023 + 6 - e) << 52);
  uint8_t* rb = rec[warp];
  double next = row[lane];  // the block's value, loaded one block ahead
  for (int64_t b = 0; b * 32 < ncols; ++b) {
    double y = next * scale;  // |y| < 64
    if ((b + 1) * 32 < ncols) next = row[(b + 1) * 32 + lane];
#pragma unroll
    for (int s = 0; s < kOzSlices; ++s) {
      int low;
      const double rr = round_shift(y, &low);
      rb[s * 32 + lane] = (uint8_t)(low & 0xFF);
      y = (y - rr) * 128.0;
    }
    rb[7 * 32 + lane] = 0;
    __syncwarp();
    if (lane < 16) {
      int8_t* dst;
      if (tile_rows == 0) {
        dst = q + r * lq + b * kOzRecord + lane * 16;
      } else if (tile_rows < 0) {
        // tiled (R'^T of the final W, -tile_rows = kp rows per subject): per
        // (subject, k-block, 64-row half) the eight slots of 64 rows x 32 B, contiguous
        // and already in TMA SWIZZLE_32B order (16-byte chunk h of row r at h ^ ((r >> 2) & 1)),
        // so the B operand of a k-block is one bulk copy instead of 64 x slots 32-byte rows
        const int64_t kpr = -tile_rows, i = r / kpr, f = r - i * kpr;
        const int64_t nz = (kpr + 63) / 64, nub = ncols / 32, rr = f & 63;
        dst = q + ((i * nub + b) * nz + (f >> 6)) * kOzRTile + (lane >> 1) * 2048 + rr * 32 +
              (((lane & 1) ^ ((rr >> 2) & 1)) << 4);
      } else {
        // tiled (G_i): record halves of 128 rows x one k-block contiguous
        const int64_t i = r / tile_rows, t = r - i * tile_rows;
        const int64_t ntb = (tile_rows + 127) / 128, nub = ncols / 32;
        dst = q + ((i * ntb + t / 128) * nub + b) * (2 * kOzBox) + (lane >> 3) * kOzBox + (t & 127) * 128 + (lane & 7) * 16;
      }
      *reinterpret_cast<uint4*>(dst) = reinterpret_cast<const uint4*>(rb)[lane];
    }
    __syncwarp();
  }
}

// the same slices for a few long rows (S: kp rows, every iteration): one CTA
// of eight warps per row, the row maximum by a block reduction and the
// 32-column blocks spread over the warps (plain layout only)
__global__ void __launch_bounds__(256) k_oz_slice_rows_wide(const double* __restrict__ M, int64_t ldm,
                                                            int64_t ncols, int8_t* __restrict__ q, int64_t lq,
                                                            int32_t* __restrict__ expo) {
  __shared__ __align__(16) uint8_t rec[8][kOzRecord];
  __shared__ double wmax[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x;
  const double* row = M + r * ldm;
  double m = 0.0;
  for (int64_t c = threadIdx.x; c < ncols; c += 256) m = fmax(m, fabs(row[c]));
  m = warp_max(m);
  if (lane == 0) wmax[warp] = m;
  __syncthreads();
  m = wmax[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m = fmax(m, wmax[w]);
  const int e = (m > 0.0) ? frexp_exp(m) : 0;
  if (threadIdx.x == 0) expo[r] = e;
  const double scale = __longlong_as_double((long long)(1023 + 6 - e) << 52);
  uint8_t* rb = rec[warp];
  for (int64_t b = warp; b * 32 < ncols; b += 8) {
    double y = row[b * 32 + lane] * scale;  // |y| < 64
#pragma unroll
    for (int s = 0; s < kOzSlices; ++s) {
      int low;
      const double rr = round_shift(y, &low);
      rb[s * 32 + lane] = (uint8_t)(low & 0xFF);
      y = (y - rr) * 128.0;
    }
    rb[7 * 32 + lane] = 0;
    __syncwarp();
    if (lane < 16) reinterpret_cast<uint4*>(q + r * lq + b * kOzRecord)[lane] = reinterpret_cast<const uint4*>(rb)[lane];
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// B_i = S G_i / 2 from the slices: CTA = (128 TRs t of subject i) x all 64
// features f, contraction over the TRs u of G_i's rows in 32-wide blocks:
//   B^T[t][f] = 1/2 sum_u G[t][u] S[f][u]
//             = 1/2 2^{e_t + s_f} sum_d 2^{-12-7d} sum_{s+s'=d} (Qg_s Qs_{s'}^T)[t][f]
// tcgen05.mma kind::i8 M = 128 (t), N = 64 (f), K = 32; all seven d-groups
// accumulate in TMEM at once (7 x 64 columns), one pass; the epilogue writes
// B[f][t] (coalesced over t) into the reduced record bred[i].
//
// The same kernel (kRowW) forms the model's W_i = Xhat_i R_i at the end of a
// Gram-path fit, with R_i = S^T M_i / 2 (srm.py:147 + kernels.py:212 via
// W = A M): A = the voxel-major slices Qt of Xhat (rows = voxels, K = TRs),
// B = the row slices of R'^T = (2^{e_t} R_i)^T (the column scales of Xhat
// folded into R), so W[v][f] = 2^{r_f} sum_d 2^{-12-7d} (...)[v][f].
// ---------------------------------------------------------------------------
constexpr int kSgStages = 4;
// kRowWX: the final W of four-slice (fp32) X-hat with the A operand sliced in
// the kernel from X-hat itself: TMA brings 128 voxels x 32 TRs of fp32 as
// 128-byte rows (the records' 32-byte voxel runs bound kRowW by TMA row issue,
// ~0.3 of HBM), four slicer warps cut them into the same int8 digits the
// records hold (k_oz_split_f32's N = rint(x 2^(27 - e_t)), balanced base-128)
// and write them K-major (SWIZZLE_32B, the layout TMA gives the B operand), so
// the MMAs and the result are kRowW's bit for bit
enum RowGemmMode { kRowSG = 0, kRowW = 1, kRowWX = 2 };

// Per-stage shared memory of k_oz_rowgemm<MODE, NSA, ND>: the A boxes (kRowSG:
// the G record halves holding the slices used; kRowW: NSA MN-major slices of
// 128 voxels x 32 TRs) and the B record halves.  ND = 7 d-groups take 448 of
// the 512 TMEM columns (one CTA per SM); ND = 4 (four-slice operands, pairs
// s + s' >= 4 dropped) takes 256 and two CTAs share an SM.
template <int MODE, int NSA, int ND>
struct RowGemmShape {
  static constexpr int halves = ND > 4 ? 2 : 1;
  static constexpr int a_bytes = MODE == kRowSG ? halves * kOzBox : NSA * 4096;
  // kRowWX: the fp32 X-hat tile ahead of the slices (128 rows x 128 B, SWIZZLE_128B)
  static constexpr int x_bytes = MODE == kRowWX ? 128 * 32 * 4 : 0;
  // B: the slots of 64 rows x 32 B (k-block of 32 TRs), slot-major -- all
  // eight, or for kRowW with ND <= 6 the six its slot pairs (s2, s2 + 1),
  // s2 <= ND - 2, read (the map's box must match: make_map_q8 slots)
  static constexpr int b_slots = (MODE != kRowSG && ND <= 6) ? 6 : 8;
  static constexpr int b_bytes = b_slots * 64 * 32;
  static constexpr int stage_bytes = x_bytes + a_bytes + b_bytes;
  // kRowW keeps a W staging tile (128 rows x 64 features, pitch 65) beside the
  // ring: three stages of seven-slice operands fit with it, four otherwise
  static constexpr int stages = ((MODE == kRowW && NSA > 4) || MODE == kRowWX) ? 3 : kSgStages;
  static constexpr int wst_pitch = 65;
  static constexpr int wst_bytes = MODE != kRowSG ? 128 * wst_pitch * 8 : 0;
  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue; kRowWX: warps 10-13 slice
  static constexpr int threads = MODE == kRowWX ? 448 : 320;
  static constexpr uint32_t tmem_cols = 512;  // eight 64-column d-groups (d = 7 unused)
  static constexpr int ctas_per_sm = 1;
  static constexpr size_t smem_bytes = (size_t)stages * stage_bytes + wst_bytes + 1024;
};

struct RowGemmArgs {
  const int32_t* aexp;   // kRowSG: G row exponents [n_local][ldx]
  const int32_t* bexp;   // kRowSG: S row exponents [kp]; kRowW: R'^T row exponents [n_local][kp]
  double* out;           // kRowSG: bred; kRowW: W [rows_total][K]
  const OzItem* items;   // kRowW: {subject, local voxel v0, global row of v0, valid rows}
  const int8_t* bt;      // kRowW / kRowWX: the tiled R'^T slices (k_oz_slice_rows, tile_rows < 0)
  int64_t ldx, kp, ldo, K;
  int first;             // kRowSG: subject of the first tile
  int n_work;            // tiles: kRowSG (subject, 128-TR block, feature half); kRowW (item, feature half)
  int nz, ntb;           // feature halves; kRowSG: 128-TR blocks per subject
  int zseq;              // kRowW / kRowWX: a CTA takes every feature half of its items, one after the other
};

// the operands of work tile w: subject, first A row, feature half
struct RowTile {
  int i, arow, z, nvb;
  int64_t n0;
};

template <int MODE>
__device__ __forceinline__ RowTile row_tile(const RowGemmArgs& g, int w) {
  RowTile r;
  r.z = w % g.nz;
  if (MODE == kRowSG) {
    const int tb = (w / g.nz) % g.ntb;
    r.i = g.first + w / (g.nz * g.ntb);
    r.arow = tb * 128;
    r.nvb = 128;
    r.n0 = 0;
  } else {
    const OzItem it = g.items[w / g.nz];
    r.i = it.subj;
    r.arow = it.m0;
    r.nvb = it.nvb;
    r.n0 = it.n0;
  }
  return r;
}

// The j-th work tile of this CTA (>= n_work: none left; increasing in j).
// zseq: items c, c + grid, ... with their nz feature halves back to back on
// the same CTA, so the second half's A operand is an L2 hit on this SM's own
// L2 partition (halves on neighbouring CTAs land on either die: ncu showed
// 1.7x the A bytes from DRAM at kp = 128)
__device__ __forceinline__ int row_work(const RowGemmArgs& g, int j) {
  if (!g.zseq) return (int)blockIdx.x + j * (int)gridDim.x;
  return ((j / g.nz) * (int)gridDim.x + (int)blockIdx.x) * g.nz + j % g.nz;
}

// Row GEMM CTAs: warp 0 TMA producer, warp 1 MMA issuer, warps 2-9 epilogue
// (two warps per TMEM lane quarter, each on 32 of the 64 columns: the
// epilogue is latency-bound, and its TMEM release gates the next tile's MMAs)
constexpr int kRowThreads = 320;
constexpr int kRowEpi = kRowThreads - 64;

// Seven d-groups of 8 accumulator columns -> two exact int64 partial sums
//   H = sum_{d<4} raw_d 2^{7(3-d)},  L = sum_{d>=4} raw_d 2^{7(6-d)}
// (|raw| < 2^31: |H| < 2^53, |L| < 2^46), so that
//   sum_d raw_d 2^{-12-7d} = H 2^-33 + L 2^-54
// is formed with two exact conversions and one rounding (oz_hl_value).  H and
// L are linear in the accumulators: parts of a split contraction add exactly.
// ND < 7: the d-groups beyond ND - 1 count as zero (an N = 128 MMA may have
// written a partial group ND; it is not read)
template <int ND = 7>
__device__ __forceinline__ void oz_load_hl(uint32_t taddr, long long* H, long long* L) {
  uint32_t raw[7][8];
#pragma unroll
  for (int d = 0; d < 7; ++d) {
    if (d < ND)
      tmem_ld8(taddr + 64u * (uint32_t)d, raw[d]);
    else
#pragma unroll
      for (int j = 0; j < 8; ++j) raw[d][j] = 0u;
  }
  tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    // (multiplications, not shifts: the sums are signed)
    H[j] = (long long)(int32_t)raw[0][j] * (1LL << 21) + (long long)(int32_t)raw[1][j] * (1LL << 14) +
           (long long)(int32_t)raw[2][j] * 128 + (long long)(int32_t)raw[3][j];
    L[j] = (long long)(int32_t)raw[4][j] * (1LL << 14) + (long long)(int32_t)raw[5][j] * 128 + (long long)(int32_t)raw[6][j];
  }
}

__device__ __forceinline__ double oz_hl_value(long long H, long long L) {
  return fma((double)L, 0x1p-54, (double)H * 0x1p-33);
}

// NSA: slices of the A operand (kRowW: X-hat's 7 or 4; kRowSG: G's 7).
// ND: d-groups kept (all 7 in the current uses).  Persistent: CTA c takes
// work tiles c, c + gridDim.x, ...; the producer streams the next tile's
// k-blocks while the epilogue drains the last, and the MMA warp waits only
// for the accumulators to be drained (accempty).
template <int MODE, int NSA, int ND>
__global__ void __launch_bounds__(RowGemmShape<MODE, NSA, ND>::threads, RowGemmShape<MODE, NSA, ND>::ctas_per_sm)
    k_oz_rowgemm(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, RowGemmArgs g) {
  using Shape = RowGemmShape<MODE, NSA, ND>;
  constexpr int kStage = Shape::stage_bytes;
  constexpr int kSt = Shape::stages;
  extern __shared__ __align__(1024) unsigned char oz_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kSt], empty[kSt], sliced[kSt], accfull, accempty;
  __shared__ uint32_t tmem_base;
  const int64_t ldx = g.ldx, kp = g.kp, ldo = g.ldo;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nub = (int)(ldx / 32);
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < kSt; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
        mbar_init(&sliced[s], 4);  // kRowWX: one arrival per slicer warp
      }
      mbar_init(&accfull, 1);
      mbar_init(&accempty, kRowEpi / 32);
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
  } else if (warp == 1) {
    tmem_alloc(&tmem_base, Shape::tmem_cols);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (warp == 0) {
    if (lane == 0) {
      int kk = 0;
      for (int j = 0, w = row_work(g, 0); w < g.n_work; w = row_work(g, ++j)) {
        const RowTile tl = row_tile<MODE>(g, w);
        for (int k = 0; k < nub; ++k, ++kk) {
          const int slot = kk % kSt;
          if (kk >= kSt) mbar_wait(&empty[slot], ((kk / kSt) - 1) & 1);
          unsigned char* st = smem + slot * kStage;
          mbar_expect_tx(&full[slot], (uint32_t)(MODE == kRowWX ? kStage - Shape::a_bytes : kStage));
          if (MODE == kRowWX) {
            // fp32 X-hat rows v0 .. v0 + 127 (global), TRs 32 k .. 32 k + 31
            tma_load_2d(st, &tma, k * 32, tl.n0, &full[slot]);
          } else if (MODE == kRowSG) {
            // tiled G slices: (128-row block, k-block, record half) rows of 128 B
            const int grow = ((tl.arow / 128) * nub + k) * 256;
            tma_load_3d(st, &tma, 0, grow, tl.i, &full[slot]);
            if (Shape::halves > 1) tma_load_3d(st + kOzBox, &tma, 0, grow + 128, tl.i, &full[slot]);
          } else {
            // Q records of 32 TRs x 4 voxel blocks x nsa slots -> [slot][vb][t][32 B]
            tma_load_5d(st, &tma, 0, k * 32, tl.arow / 32, 0, tl.i, &full[slot]);
          }
          if (MODE == kRowSG)
            tma_load_4d(st + Shape::x_bytes + Shape::a_bytes, &tmb, 0, tl.z * 64, k * 8, 0, &full[slot]);
          else  // one contiguous run of the slots read, already in the SWIZZLE_32B order
            bulk_load(st + Shape::x_bytes + Shape::a_bytes,
                      g.bt + (((int64_t)tl.i * nub + k) * g.nz + tl.z) * kOzRTile, (uint32_t)Shape::b_bytes, &full[slot]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kRowW: A (voxels x TRs) is MN-major (bit 15): voxels contiguous in the Q records.
      // N = 128: B is the slot pair (s2, s2 + 1) of 64 features each, so one MMA
      // feeds d-groups s + s2 and s + s2 + 1 (adjacent 64-column accumulators);
      // an N = 64 MMA costs the same tensor-pipe time as N = 128 (tools/i8_peak.cu)
      constexpr uint32_t idesc = idesc_s8(128, 128) | (MODE == kRowW ? (1u << 15) : 0u);  // kRowWX: A K-major
      int kk = 0, li = 0;
      for (int w = row_work(g, 0); w < g.n_work; w = row_work(g, ++li)) {
        if (li > 0) mbar_wait(&accempty, (li - 1) & 1);  // the last tile's accumulators drained
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int k = 0; k < nub; ++k, ++kk) {
          const int slot = kk % kSt;
          mbar_wait(MODE == kRowWX ? &sliced[slot] : &full[slot], (kk / kSt) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(smem + slot * kStage + Shape::x_bytes);
          const uint32_t sb = sa + Shape::a_bytes;
          // one descriptor per operand and stage; a slice is a constant offset of
          // the 16-byte address field (no carry: smem addresses < 2^18)
          const uint64_t da0 = MODE == kRowSG   ? umma_desc_sw128(sa)
                               : MODE == kRowW  ? umma_desc_sw32_mn(sa, 1024, 256)
                                                : umma_desc_sw32_mn(sa, 16, 256);  // kRowWX: K-major, as B
          // K-major SWIZZLE_32B: 8-row atoms of 256 B (SBO); slot j starts at 2 KB j
          const uint64_t db0 = umma_desc_sw32_mn(sb, 16, 256);
          const uint32_t keep = k == 0 ? 0u : 1u;
          // s = 0 first: its four pairs cover all eight d-groups once, so they alone
          // start the accumulators of a fresh tile
#pragma unroll
          for (int s = 0; s < NSA; ++s) {
            const uint64_t aoff = MODE == kRowSG ? (uint64_t)((s >> 2) * (kOzBox >> 4) + 2 * (s & 3))
                                                 : (uint64_t)(s * (4096 >> 4));
#pragma unroll
            for (int s2 = 0; s2 + s <= ND - 1; s2 += 2)
              mma_s8(tmem + 64u * (uint32_t)(s + s2), da0 + aoff, db0 + (uint64_t)(s2 * (2048 >> 4)), idesc,
                     s == 0 ? keep : 1u);
          }
          mma_commit(&empty[slot]);
        }
        mma_commit(&accfull);
      }
    }
  } else if (MODE == kRowWX && warp >= 10) {
    // ---------------- slicers (kRowWX): thread r cuts voxel row r of the tile ----------------
    const int r = (int)threadIdx.x - 320;
    int kk = 0;
    for (int j = 0, w = row_work(g, 0); w < g.n_work; w = row_work(g, ++j)) {
      const RowTile tl = row_tile<MODE>(g, w);
      const int32_t* ex = g.aexp + (int64_t)tl.i * ldx;  // X-hat column exponents e_t (k_oz_split_f32's)
      for (int k = 0; k < nub; ++k, ++kk) {
        const int slot = kk % kSt;
        int e[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) e[j] = __ldg(ex + k * 32 + j);
        mbar_wait(&full[slot], (kk / kSt) & 1);
        const unsigned char* xs = smem + slot * kStage;  // [128 rows][128 B], SWIZZLE_128B
        unsigned char* as = smem + slot * kStage + Shape::x_bytes;
        uint32_t wd[4][8];  // [slice][four TRs per word]
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          // 16-byte chunk c of row r sits at chunk c ^ (r & 7)
          const float4 q = *reinterpret_cast<const float4*>(xs + r * 128 + ((c ^ (r & 7)) << 4));
          const float xv[4] = {q.x, q.y, q.z, q.w};
          int dg[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int ej = e[4 * c + u];
            int n;
            if (ej >= -100 && ej <= 153)
              n = __float2int_rn(xv[u] * __int_as_float((127 + 27 - ej) << 23));
            else
              n = __double2int_rn((double)xv[u] * ldexp(1.0, 27 - ej));
#pragma unroll
            for (int sl = 3; sl >= 1; --sl) {
              const int n1 = (n + 64) >> 7;
              dg[sl][u] = n - (n1 << 7);
              n = n1;
            }
            dg[0][u] = n;
          }
#pragma unroll
          for (int sl = 0; sl < 4; ++sl) {
            const uint32_t lo = __byte_perm((uint32_t)dg[sl][0], (uint32_t)dg[sl][1], 0x0040);
            const uint32_t hi = __byte_perm((uint32_t)dg[sl][2], (uint32_t)dg[sl][3], 0x0040);
            wd[sl][c] = __byte_perm(lo, hi, 0x5410);
          }
        }
        // slice sl, row r: 32 bytes (TRs 0-31) as two 16-byte chunks, chunk h at h ^ ((r >> 2) & 1)
        // (TMA SWIZZLE_32B's layout of 32-byte rows)
#pragma unroll
        for (int sl = 0; sl < 4; ++sl)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            *reinterpret_cast<uint4*>(as + sl * 4096 + r * 32 + ((h ^ ((r >> 2) & 1)) << 4)) =
                make_uint4(wd[sl][4 * h], wd[sl][4 * h + 1], wd[sl][4 * h + 2], wd[sl][4 * h + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tcgen05 reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&sliced[slot]);
      }
    }
  } else {
    static_assert(ND >= 5 && ND <= 7, "the H/L epilogue combines d-groups 0-3 and 4-6");
    const int quarter = warp & 3;              // TMEM lanes 32 quarter .. + 31 (warp % 4)
    const int cbase = ((warp - 2) >> 2) * 32;  // this warp's 32 of the 64 columns
    const int r = quarter * 32 + lane;
    const int etid = (warp - 2) * 32 + lane;
    double* wst = reinterpret_cast<double*>(smem + kSt * kStage);  // kRowW staging tile
    const int fmax_ = MODE == kRowSG ? (int)kp : (int)g.K;
    const int half = MODE == kRowSG ? -1 : 0;  // the 1/2 of B = S G / 2 (R already holds its 1/2)
    int li = 0;
    for (int w = row_work(g, 0); w < g.n_work; w = row_work(g, ++li)) {
      const RowTile tl = row_tile<MODE>(g, w);
      const int f0 = tl.z * 64;
      // kRowSG: B[f][t] of subject i; kRowW: W[row][f]
      const int64_t t = tl.arow + r;
      const bool valid = MODE == kRowSG ? t < ldx : r < tl.nvb;
      const int32_t* bexp = MODE == kRowSG ? g.bexp : g.bexp + (int64_t)tl.i * kp;
      // scale exponents ahead of the accumulators
      const int et = (MODE == kRowSG && valid) ? __ldg(g.aexp + (int64_t)tl.i * ldx + t) : 0;
      int be[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) be[j] = (f0 + cbase + j < fmax_) ? __ldg(bexp + f0 + cbase + j) : 0;
      mbar_wait(&accfull, li & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      double* out = MODE == kRowSG ? g.out + (int64_t)tl.i * kp * ldo + t : wst + r * Shape::wst_pitch;
      const int64_t fstride = MODE == kRowSG ? ldo : 1;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int c0 = cbase + 8 * c;
        long long H[8], L[8];
        oz_load_hl<ND>(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, H, L);
        if (valid) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int f = f0 + c0 + j;
            if (f < fmax_)
              out[(int64_t)(MODE == kRowSG ? f : c0 + j) * fstride] = oz_hl_value(H[j], L[j]) * pow2(et + be[8 * c + j] + half);
          }
        }
      }
      // accumulators drained: the MMA warp may start the next tile
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty);
      if (MODE != kRowSG) {
        asm volatile("bar.sync 1, %0;" ::"r"(kRowEpi) : "memory");  // the staged tile is complete
        const int K = (int)g.K;
        const int nc = min(64, K - f0);  // this tile's columns f0 .. f0 + nc - 1 of W
        double* dst = g.out + tl.n0 * K + f0;
        for (int e = etid; e < tl.nvb * nc; e += kRowEpi)
          dst[(int64_t)(e / nc) * K + e % nc] = wst[(e / nc) * Shape::wst_pitch + e % nc];
        asm volatile("bar.sync 1, %0;" ::"r"(kRowEpi) : "memory");  // staging free for the next tile
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) tmem_free(tmem, Shape::tmem_cols);
}

// ---------------------------------------------------------------------------
// B_i = S G_i / 2, stream-K: the (subject, 128-TR block, 64-feature half)
// tiles of all subjects laid end to end as one run of 32-TR k-blocks, and
// persistent CTA c (one per SM, a few SMs left to the side lane's one-CTA
// tail kernels) takes k-blocks [c L, (c + 1) L), L >= a tile's k-blocks, so
// every CTA does the same number of MMAs (the per-tile grid ran 2.2 waves of
// 320 CTAs in 3) and the next tile's TMA loads run under the epilogue.
//
// A tile cut by a range boundary has two parts: its tail (first segment of
// CTA c + 1) parks its raw int32 d-group sums in part[c + 1] and raises
// flag[c + 1]; its head (last segment of CTA c) waits for the flag, adds the
// parked sums in int32 -- exact, so B_i is bit-identical to the per-tile
// kernel's for any split, shard layout or SM count -- and stores the tile.
// Same MMAs, TMEM layout and epilogue arithmetic as k_oz_rowgemm<kRowSG>.
// ---------------------------------------------------------------------------
constexpr int kSkParkPairs = 64 * 128;  // (H, L) per (feature, TR) of a tile

struct SkArgs {
  const int32_t* aexp;  // G row exponents [n_local][ldx]
  const int32_t* bexp;  // S row exponents [kp]
  double* out;          // bred
  long long* part;      // [grid][2][kSkParkPairs]: parked (H, L) of a tile's tail
  int32_t* flag;        // [grid], zero between launches
  int64_t ldx, kp, ldo;
  int first;            // subject of the first tile
  int ntb, nz, nub;     // TR blocks per subject, feature halves, k-blocks per tile
  int64_t units, span;  // total k-blocks, k-blocks per CTA
};

// the tile and k-block range [kb0, kb1) of the segment starting at unit u
__device__ __forceinline__ void sk_segment(const SkArgs& g, int64_t u, int64_t u1, int* tile, int* kb0, int* kb1) {
  *tile = (int)(u / g.nub);
  *kb0 = (int)(u - (int64_t)*tile * g.nub);
  *kb1 = (int)(u1 - u < (int64_t)(g.nub - *kb0) ? *kb0 + (u1 - u) : g.nub);
}

__global__ void __launch_bounds__(kRowThreads, 1)
    k_oz_sg_sk(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, SkArgs g) {
  using Shape = RowGemmShape<kRowSG, kOzSlices, 7>;
  constexpr int kStage = Shape::stage_bytes;
  constexpr int ND = 7;
  extern __shared__ __align__(1024) unsigned char oz_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kSgStages], empty[kSgStages], accfull, accempty;
  __shared__ uint32_t tmem_base;
  const int64_t u_begin = (int64_t)blockIdx.x * g.span;
  const int64_t u_end = min(g.units, u_begin + g.span);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < kSgStages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      mbar_init(&accfull, 1);
      mbar_init(&accempty, kRowEpi / 32);  // one arrive per epilogue warp
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
  } else if (warp == 1) {
    tmem_alloc(&tmem_base, Shape::tmem_cols);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      for (int64_t u = u_begin; u < u_end; ++u, ++k) {
        const int tile = (int)(u / g.nub), kb = (int)(u - (int64_t)tile * g.nub);
        const int z = tile % g.nz, tb = (tile / g.nz) % g.ntb, i = g.first + tile / (g.nz * g.ntb);
        const int slot = k % kSgStages;
        if (k >= kSgStages) mbar_wait(&empty[slot], ((k / kSgStages) - 1) & 1);
        unsigned char* st = smem + slot * kStage;
        mbar_expect_tx(&full[slot], (uint32_t)kStage);
        const int grow = (tb * g.nub + kb) * 256;  // tiled G slices
        tma_load_3d(st, &tma, 0, grow, i, &full[slot]);
        tma_load_3d(st + kOzBox, &tma, 0, grow + 128, i, &full[slot]);
        tma_load_4d(st + Shape::a_bytes, &tmb, 0, z * 64, kb * 8, 0, &full[slot]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_s8(128, 128);
      int k = 0, seg = 0;
      for (int64_t u = u_begin; u < u_end; ++seg) {
        int tile, kb0, kb1;
        sk_segment(g, u, u_end, &tile, &kb0, &kb1);
        // the epilogue has drained the previous segment's accumulators
        if (seg > 0) mbar_wait(&accempty, (seg - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int kb = kb0; kb < kb1; ++kb, ++k) {
          const int slot = k % kSgStages;
          mbar_wait(&full[slot], (k / kSgStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(smem + slot * kStage);
          const uint64_t da0 = umma_desc_sw128(sa);
          const uint64_t db0 = umma_desc_sw32_mn(sa + Shape::a_bytes, 16, 256);
          const uint32_t keep = kb == kb0 ? 0u : 1u;
#pragma unroll
          for (int s = 0; s < kOzSlices; ++s) {
            const uint64_t aoff = (uint64_t)((s >> 2) * (kOzBox >> 4) + 2 * (s & 3));
#pragma unroll
            for (int s2 = 0; s2 + s <= ND - 1; s2 += 2)
              mma_s8(tmem + 64u * (uint32_t)(s + s2), da0 + aoff, db0 + (uint64_t)(s2 * (2048 >> 4)), idesc,
                     s == 0 ? keep : 1u);
          }
          mma_commit(&empty[slot]);
        }
        mma_commit(&accfull);
        u += kb1 - kb0;
      }
    }
  } else {
    const int quarter = warp & 3;
    const int cbase = ((warp - 2) >> 2) * 32;
    const int r = quarter * 32 + lane;
    const int etid = (warp - 2) * 32 + lane;  // 0 .. kRowEpi - 1
    int seg = 0;
    for (int64_t u = u_begin; u < u_end; ++seg) {
      int tile, kb0, kb1;
      sk_segment(g, u, u_end, &tile, &kb0, &kb1);
      u += kb1 - kb0;
      const int z = tile % g.nz, tb = (tile / g.nz) % g.ntb, i = g.first + tile / (g.nz * g.ntb);
      const bool tail = kb0 > 0;      // park for the previous CTA
      const bool head = kb1 < g.nub;  // finish with the next CTA's parked part
      // scale exponents ahead of the accumulators
      const int f0 = z * 64;
      const int64_t t = (int64_t)tb * 128 + r;
      const bool valid = t < g.ldx;
      const int et = (valid && !tail) ? __ldg(g.aexp + (int64_t)i * g.ldx + t) : 0;
      int be[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) be[j] = (!tail && f0 + cbase + j < g.kp) ? __ldg(g.bexp + f0 + cbase + j) : 0;
      mbar_wait(&accfull, seg & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      long long* pout = g.part + (int64_t)blockIdx.x * 2 * kSkParkPairs;
      const long long* pin = g.part + (int64_t)(blockIdx.x + 1) * 2 * kSkParkPairs;
      if (tail) {
        // drain and park (the stores do not hold the warp), then release
#pragma unroll 1
        for (int c0 = cbase; c0 < cbase + 32; c0 += 8) {
          long long H[8], L[8];
          oz_load_hl(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, H, L);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            pout[(c0 + j) * 128 + r] = H[j];
            pout[kSkParkPairs + (c0 + j) * 128 + r] = L[j];
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&accempty);
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"r"(kRowEpi) : "memory");
        if (etid == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(g.flag + blockIdx.x), "r"(1) : "memory");
        continue;
      }
      if (head) {
        // the next CTA parks this tile's tail first thing in its range
        if (etid == 0) {
          const int32_t* fl = g.flag + blockIdx.x + 1;
          int v = 0;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
          } while (v == 0);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kRowEpi) : "memory");
      }
      double* out = g.out + (int64_t)i * g.kp * g.ldo + t;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int c0 = cbase + 8 * c;
        // the parked part: all sixteen L2 loads in flight before the TMEM drain
        // (ld.global.cg: the lines may be cached nowhere but L2)
        long long ph[8], pl[8];
        if (head) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(ph[j]) : "l"(pin + (c0 + j) * 128 + r));
            asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(pl[j]) : "l"(pin + kSkParkPairs + (c0 + j) * 128 + r));
          }
        }
        long long H[8], L[8];
        oz_load_hl(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, H, L);
        if (head) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            H[j] += ph[j];
            L[j] += pl[j];
          }
        }
        if (valid) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int f = f0 + c0 + j;
            if (f < g.kp) out[(int64_t)f * g.ldo] = oz_hl_value(H[j], L[j]) * pow2(et + be[8 * c + j] - 1);
          }
        }
      }
      // accumulators drained: the MMA warp may start the next segment
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty);
      if (head && etid == 0) g.flag[blockIdx.x + 1] = 0;  // consumed: ready for the next launch
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) tmem_free(tmem, Shape::tmem_cols);
}

// R'^T[i][f][t] = 2^{e_t} (M_i^T S)[f][t] / 2 for the final W = Xhat R
// (M_i = mmat[i], kp x kp; S = kp x ldx); one thread per (f, t), subject = blockIdx.y
__global__ void __launch_bounds__(256) k_oz_rt(const double* __restrict__ mmat, const double* __restrict__ S,
                                               const int32_t* __restrict__ expo, double* __restrict__ rt,
                                               int64_t ldx, int64_t kp, int64_t K) {
  const int i = blockIdx.y;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= kp * ldx) return;
  const int64_t f = e / ldx, t = e - f * ldx;
  const double* M = mmat + (int64_t)i * kp * kp;
  double s = 0.0;
  if (f < K)
    for (int64_t c = 0; c < K; ++c) s += M[c * kp + f] * S[c * ldx + t];
  rt[(int64_t)i * kp * ldx + e] = s * pow2(expo[(int64_t)i * ldx + t] - 1);
}

}  // namespace

size_t oz_gram_smem_bytes() { return (size_t)kOzStages * kOzStageBytes + 1024; }

size_t oz_tiled_bytes(int64_t rows, int64_t ncols) { return (size_t)((rows + 127) / 128) * (ncols / 32) * 2 * kOzBox; }

cudaError_t launch_oz_slice_rows(const double* M, int64_t ldm, int64_t rows, int64_t ncols, int8_t* q, int64_t lq,
                                 int32_t* expo, cudaStream_t st, int64_t tile_rows) {
  if (rows <= 0) return cudaSuccess;
  if (ncols % 32 != 0) return cudaErrorInvalidValue;
  if (tile_rows == 0 && rows <= 1024)  // (the tiled layouts go through k_oz_slice_rows)
    k_oz_slice_rows_wide<<<(unsigned)rows, 256, 0, st>>>(M, ldm, ncols, q, lq, expo);
  else
    k_oz_slice_rows<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(M, ldm, rows, ncols, q, lq, expo, tile_rows);
  return cudaGetLastError();
}

namespace {

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        n <= 0) {
      cudaGetLastError();
      n = 148;
    }
  }
  return n;
}

// max_ctas > 0: persistent grid of at most max_ctas CTAs; else one CTA per tile
template <int MODE, int NSA, int ND>
cudaError_t run_rowgemm(const TmaMap& ta, const TmaMap& tb, RowGemmArgs g, int max_ctas, cudaStream_t st) {
  const size_t bytes = RowGemmShape<MODE, NSA, ND>::smem_bytes;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(k_oz_rowgemm<MODE, NSA, ND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (g.n_work <= 0) return cudaSuccess;
  if (g.kp > 128 || g.ldx % 32 != 0) return cudaErrorInvalidValue;
  // persistent kRowW / kRowWX grids with two feature halves: both halves of an item on one CTA
  // (SRM_B200_OZW_ZSEQ=0 restores halves on neighbouring CTAs; same tiles, bit-identical W)
  const char* zenv = getenv("SRM_B200_OZW_ZSEQ");  // (read per launch: the tests toggle it)
  const bool zseq_on = !(zenv && zenv[0] == '0');
  g.zseq = (MODE != kRowSG && g.nz > 1 && max_ctas > 0 && zseq_on) ? 1 : 0;
  const int units = g.zseq ? g.n_work / g.nz : g.n_work;
  const int grid = max_ctas > 0 ? std::min(units, max_ctas) : g.n_work;
  k_oz_rowgemm<MODE, NSA, ND><<<grid, RowGemmShape<MODE, NSA, ND>::threads, bytes, st>>>(*reinterpret_cast<const CUtensorMap*>(ta.opaque),
                                                               *reinterpret_cast<const CUtensorMap*>(tb.opaque), g);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_oz_sg(const TmaMap& tmg, const TmaMap& tms, const int32_t* gexp, const int32_t* sexp,
                         double* bred, int64_t ldx, int64_t kp, int64_t ldo, int first, int count, cudaStream_t st) {
  RowGemmArgs g{gexp, sexp, bred, nullptr, nullptr, ldx, kp, ldo, 0, first, 0, (int)((kp + 63) / 64), (int)((ldx + 127) / 128)};
  g.n_work = count * g.nz * g.ntb;
  return run_rowgemm<kRowSG, kOzSlices, 7>(tmg, tms, g, 0, st);
}

size_t oz_sk_park_bytes() { return (size_t)kSkParkPairs * 16; }

cudaError_t launch_oz_sg_sk(const TmaMap& tmg, const TmaMap& tms, const int32_t* gexp, const int32_t* sexp,
                            double* bred, int32_t* part, int32_t* flag, int64_t ldx, int64_t kp, int64_t ldo,
                            int first, int count, int max_ctas, cudaStream_t st) {
  using Shape = RowGemmShape<kRowSG, kOzSlices, 7>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_oz_sg_sk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Shape::smem_bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (count <= 0) return cudaSuccess;
  if (kp > 128 || ldx % 32 != 0 || max_ctas <= 0) return cudaErrorInvalidValue;
  SkArgs g{gexp, sexp, bred, reinterpret_cast<long long*>(part), flag, ldx, kp, ldo, first, 0, 0, 0, 0, 0};
  g.ntb = (int)((ldx + 127) / 128);
  g.nz = (int)((kp + 63) / 64);
  g.nub = (int)(ldx / 32);
  g.units = (int64_t)count * g.ntb * g.nz * g.nub;
  // at least one tile per CTA, so a tile meets at most two CTA ranges
  g.span = std::max<int64_t>(g.nub, (g.units + max_ctas - 1) / max_ctas);
  const unsigned grid = (unsigned)((g.units + g.span - 1) / g.span);
  // a head CTA spins on a flag its tail CTA raises, so every CTA of the grid
  // must be resident at once: launched cooperatively, which the driver only
  // accepts when the whole grid fits at this kernel's occupancy (checked here
  // too, so an oversized grid is an error rather than a deadlock)
  static int max_resident = 0;
  if (max_resident == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_oz_sg_sk, kRowThreads, Shape::smem_bytes);
    if (e != cudaSuccess) return e;
    max_resident = sms * per_sm;
  }
  if ((int)grid > max_resident) return cudaErrorCooperativeLaunchTooLarge;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRowThreads);
  cfg.dynamicSmemBytes = Shape::smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_oz_sg_sk, *reinterpret_cast<const CUtensorMap*>(tmg.opaque),
                            *reinterpret_cast<const CUtensorMap*>(tms.opaque), g);
}

cudaError_t launch_oz_rt(const double* mmat, const double* S, const int32_t* expo, double* rt, int64_t ldx,
                         int64_t kp, int64_t K, int n_local, cudaStream_t st) {
  if (n_local == 0) return cudaSuccess;
  const dim3 grid((unsigned)((kp * ldx + 255) / 256), (unsigned)n_local);
  k_oz_rt<<<grid, 256, 0, st>>>(mmat, S, expo, rt, ldx, kp, K);
  return cudaGetLastError();
}

cudaError_t launch_oz_w(const TmaMap& tmqt, const TmaMap& tmr, const int8_t* rt, const int32_t* rexp, double* W,
                        const OzItem* items, int n_items, int64_t ldx, int64_t kp, int64_t K, int nsl, cudaStream_t st) {
  RowGemmArgs g{nullptr, rexp, W, items, rt, ldx, kp, 0, K, 0, 0, (int)((kp + 63) / 64), 0};
  g.n_work = n_items * g.nz;
  if (nsl == 7) return run_rowgemm<kRowW, 7, 7>(tmqt, tmr, g, sm_count(), st);
  // fp32 X-hat: d-groups 0-4 (8 MMAs per k-block instead of 12).  R's slices
  // beyond the fourth carry bits the orthonormality of W needs, and d = 4
  // keeps them; the dropped d >= 5 are ~2^-35 of the column scales, below the
  // 2^-27 truncation of X-hat's own slices (tools/slice_drop_probe.py)
  if (nsl == 4) return run_rowgemm<kRowW, 4, 5>(tmqt, tmr, g, sm_count(), st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_oz_wx(const TmaMap& tmx, const TmaMap& tmr, const int8_t* rt, const int32_t* xexp,
                         const int32_t* rexp, double* W, const OzItem* items, int n_items, int64_t ldx, int64_t kp,
                         int64_t K, cudaStream_t st) {
  RowGemmArgs g{xexp, rexp, W, items, rt, ldx, kp, 0, K, 0, 0, (int)((kp + 63) / 64), 0};
  g.n_work = n_items * g.nz;
  return run_rowgemm<kRowWX, 4, 5>(tmx, tmr, g, sm_count(), st);
}

cudaError_t launch_oz_prepare(const DevPlan& p, int x_dtype, int nsl, int first, int count,
                              unsigned long long* cmax, int8_t* q, int64_t lq, int32_t* expo, int64_t max_v,
                              cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  // seven slices for fp64 X-hat, four for fp32 (the instantiated pairs)
  if (nsl != (x_dtype == SRM_F64 ? 7 : 4)) return cudaErrorInvalidValue;
  DevPlan sub = p;
  sub.subj = p.subj + (int64_t)first * kSubjCols;
  // column maxima: kept by the demean pass (k_prep) as each subject loads
  const unsigned long long* cm = cmax + (int64_t)first * p.ldx;
  int8_t* qs = q + (int64_t)first * p.ldx * lq;
  int32_t* ex = expo + (int64_t)first * p.ldx;
  const unsigned gy = (unsigned)((p.ldx + kSplitCols - 1) / kSplitCols);
  if (x_dtype == SRM_F64)
    k_oz_split<double, 7, 1><<<dim3((unsigned)(((max_v + 31) / 32 + kSplitGroups - 1) / kSplitGroups), gy, (unsigned)count),
                               256, 0, st>>>(sub, static_cast<const double*>(p.xhat), p.ldx, p.ldx, cm, qs, lq, ex,
                                             kSplitGroups);
  else {
    // four 128-byte records per column per CTA (512-byte runs, 32 loads in
    // flight per thread): 9% faster than two on cfg 4 (SRM_B200_SPLIT_NB=2 keeps two)
    static const int nb = [] {
      const char* e = getenv("SRM_B200_SPLIT_NB");
      return e && e[0] == '2' ? 2 : 4;
    }();
    if (nb == 4)
      k_oz_split_f32<4><<<dim3((unsigned)((max_v + 127) / 128), gy, (unsigned)count), 256, 0, st>>>(
          sub, static_cast<const float*>(p.xhat), cm, qs, lq, ex);
    else  // two 128-byte records per column per CTA: 256-byte runs
      k_oz_split_f32<2><<<dim3((unsigned)((max_v + 63) / 64), gy, (unsigned)count), 256, 0, st>>>(
          sub, static_cast<const float*>(p.xhat), cm, qs, lq, ex);
  }
  return cudaGetLastError();
}

namespace {

template <int NSL>
cudaError_t run_oz_gram(const TmaMap& tmq, const OzGramOut& o, const OzItem* items, int n_items, cudaStream_t st) {
  const size_t bytes = oz_gram_smem_bytes();
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_oz_gram<NSL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  k_oz_gram<NSL><<<n_items, kOzThreads, bytes, st>>>(*reinterpret_cast<const CUtensorMap*>(tmq.opaque), o, items);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_oz_init_slices(const DevPlan& p, int first, int count, int8_t* qg, int64_t lqg, int32_t* expog,
                                  unsigned long long* cmaxg, int64_t max_v, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int K = (int)p.K;
  cudaError_t e = cudaMemsetAsync(cmaxg + (int64_t)first * K, 0, (size_t)count * K * 8, st);
  if (e != cudaSuccess) return e;
  DevPlan sub = p;
  sub.sub0 = first;
  k_oz_colmax<<<dim3((unsigned)((max_v + 255) / 256), (unsigned)count), 256, 0, st>>>(sub, p.amat, p.kp, K, cmaxg);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  DevPlan sub2 = p;
  sub2.subj = p.subj + (int64_t)first * kSubjCols;
  k_oz_split<double, 7, 1><<<dim3((unsigned)((max_v + 31) / 32), (unsigned)((K + kSplitCols - 1) / kSplitCols),
                                  (unsigned)count), 256, 0, st>>>(sub2, p.amat, p.kp, K, cmaxg + (int64_t)first * K,
                                                                  qg + (int64_t)first * K * lqg, lqg,
                                                                  expog + (int64_t)first * K, 1);
  return cudaGetLastError();
}

cudaError_t launch_oz_nt(const TmaMap& tmx, const TmaMap& tmg8, const int32_t* aexp, const int32_t* bexp,
                         double* bred, int64_t ldx, int64_t kp, int64_t ldo, int64_t K, const OzItem* items, int n_items,
                         int nslx, cudaStream_t st) {
  if (nslx != 7 && nslx != 4) return cudaErrorInvalidValue;
  const int stage = (nslx > 4 ? 2 : 1) * kOzBox + 2 * 8192;
  const size_t bytes = (size_t)4 * stage + 1024;
  static bool configured[2] = {false, false};
  const void* fn = nslx == 7 ? (const void*)k_oz_nt<7> : (const void*)k_oz_nt<4>;
  if (!configured[nslx == 7]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured[nslx == 7] = true;
  }
  if (n_items == 0) return cudaSuccess;
  if (kp > 64) return cudaErrorInvalidValue;
  OzTnArgs g{aexp, bexp, bred, ldx, kp, ldo, K};
  const CUtensorMap* x = reinterpret_cast<const CUtensorMap*>(tmx.opaque);
  const CUtensorMap* gm = reinterpret_cast<const CUtensorMap*>(tmg8.opaque);
  if (nslx == 7)
    k_oz_nt<7><<<n_items, kOzThreads, bytes, st>>>(*x, *gm, g, items);
  else
    k_oz_nt<4><<<n_items, kOzThreads, bytes, st>>>(*x, *gm, g, items);
  return cudaGetLastError();
}

cudaError_t launch_oz_tn(const TmaMap& tma, const TmaMap& tmb, const int32_t* aexp, const int32_t* bexp, double* bred,
                         int64_t ldx, int64_t kp, int64_t ldo, int64_t K, const OzItem* items, int n_items, int nslb,
                         cudaStream_t st) {
  const size_t bytes = oz_gram_smem_bytes();
  static bool configured[2] = {false, false};
  const void* fn = nslb == 7 ? (const void*)k_oz_tn<7> : (const void*)k_oz_tn<4>;
  if (nslb != 7 && nslb != 4) return cudaErrorInvalidValue;
  if (!configured[nslb == 7]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured[nslb == 7] = true;
  }
  if (n_items == 0) return cudaSuccess;
  if (kp > 128) return cudaErrorInvalidValue;
  OzTnArgs g{aexp, bexp, bred, ldx, kp, ldo, K};
  const CUtensorMap* a = reinterpret_cast<const CUtensorMap*>(tma.opaque);
  const CUtensorMap* b = reinterpret_cast<const CUtensorMap*>(tmb.opaque);
  if (nslb == 7)
    k_oz_tn<7><<<n_items, kOzThreads, bytes, st>>>(*a, *b, g, items);
  else
    k_oz_tn<4><<<n_items, kOzThreads, bytes, st>>>(*a, *b, g, items);
  return cudaGetLastError();
}

size_t oz_gram2_smem_bytes() { return (size_t)kOz2Stages * kOz2StageBytes + 1024; }

cudaError_t launch_oz_gram2(const TmaMap& tmq, const TmaMap& tmqb, const OzGramOut& o, const OzItem* items,
                            int n_items, int nsl, cudaStream_t st) {
  const size_t bytes = oz_gram2_smem_bytes();
  static bool configured[2] = {false, false};
  if (nsl != 7 && nsl != 4) return cudaErrorInvalidValue;
  const void* fn = nsl == 7 ? (const void*)k_oz_gram2<7> : (const void*)k_oz_gram2<4>;
  if (!configured[nsl == 7]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured[nsl == 7] = true;
  }
  if (n_items == 0) return cudaSuccess;
  const CUtensorMap* a = reinterpret_cast<const CUtensorMap*>(tmq.opaque);
  const CUtensorMap* b = reinterpret_cast<const CUtensorMap*>(tmqb.opaque);
  if (nsl == 7)
    k_oz_gram2<7><<<2 * n_items, kOzThreads, bytes, st>>>(*a, *b, o, items);
  else
    k_oz_gram2<4><<<2 * n_items, kOzThreads, bytes, st>>>(*a, *b, o, items);
  return cudaGetLastError();
}

cudaError_t launch_oz_gram(const TmaMap& tmq, const OzGramOut& o, const OzItem* items, int n_items, int nsl,
                           cudaStream_t st) {
  if (nsl == 7) return run_oz_gram<7>(tmq, o, items, n_items, st);
  if (nsl == 4) return run_oz_gram<4>(tmq, o, items, n_items, st);
  return cudaErrorInvalidValue;
}

}  // namespace srm
