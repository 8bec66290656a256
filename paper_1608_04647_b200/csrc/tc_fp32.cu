// fp32 streaming contractions on the 5th-generation tensor cores (tcgen05).
//
// For fp32 X-hat (BASELINE cfgs 3-5) the two per-iteration passes of the
// streaming path run as 3xTF32 split-precision MMAs with fp32 accumulators in
// TMEM: x = x_hi + x_lo with x_hi = tf32(x) (top 19 bits) and x_lo = x - x_hi,
// and   x*s ~= x_hi*s_hi + x_hi*s_lo + x_lo*s_hi   (relative error ~2^-21),
// well inside the 1e-4 fp32 tolerance of BASELINE.json.
//
//   tc_apass:  A = alpha * X S^T       (srm.py:147; M = 128 voxel rows, N = NP
//              features, K = T in 32-wide stages; both operands K-major)
//   tc_bpass:  partial B = A^T X       (srm.py:151 via W = A M; contraction
//              over a V chunk; X and A tiles are transposed into the K-major
//              core layout by the same SIMT pass that splits them)
//
// Operand tiles live in shared memory in the canonical SWIZZLE_NONE K-major
// core-matrix layout (8 rows x 16 bytes per core matrix; LBO = 128 B between
// the two K cores of an MMA step, SBO between 8-row groups), described by
// sm100 UMMA smem descriptors; one elected thread issues tcgen05.mma and
// commits to an mbarrier that guards the stage's reuse.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace srm {

namespace {

using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::mbar_wait;
using tc::mma_commit;
using tc::tma_load_2d;
using tc::tmem_alloc;
using tc::tmem_free;
using tc::umma_desc_sw128;

constexpr int kTcBK = 32;  // K (contraction) elements per stage

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm100); base offset 0; SWIZZLE_NONE
  return d;
}

// kind::tf32, fp32 accumulate, K-major A and B, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// 16 fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  tc::tmem_ld16(taddr, r);
  tc::tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// K-major SWIZZLE_NONE core layout for a [rows][kTcBK] tile, in floats
__device__ __forceinline__ int kcore(int r, int k) {
  return (r >> 3) * (kTcBK * 8) + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

__host__ __device__ constexpr int tmem_cols(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256; }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// A operand from TMEM: D[tmem] (+)= A[tmem] * B[smem desc]
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t db, uint32_t idesc, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
               :: "r"(d), "r"(a), "l"(db), "r"(idesc), "r"(acc));
}

// Each thread owns one TMEM lane of one 128-row half: it writes its 32 raw
// fp32 values (the MMA reads them as tf32 = hi) and their residuals (lo) into
// the A-operand buffer at column base `col`.
__device__ __forceinline__ void store_split_row(uint32_t tmem_lane_base, uint32_t col, const float* vals) {
  uint32_t raw[16], lo[16];
#pragma unroll
  for (int half = 0; half < 2; ++half) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float x = vals[half * 16 + j];
      raw[j] = __float_as_uint(x);
      lo[j] = __float_as_uint(x - tf32_hi(x));
    }
    tmem_st16(tmem_lane_base + col + half * 16, raw);
    tmem_st16(tmem_lane_base + col + 32 + half * 16, lo);
  }
}

constexpr int kTcT = 256;            // threads: two 128-lane halves x 4 warps
constexpr int kXStride = 36;          // A-pass raw row stride (floats): 16B aligned, LDS.128 conflict-free

// TMEM columns: accumulators of the two halves at [0,128) and [128,256); A
// operand buffers b in {0,1} at 256 + 128 b + 64 h: raw [0,32), lo [32,64)
__device__ __forceinline__ uint32_t abuf_col(int b, int h) { return 256u + 128u * b + 64u * h; }

// Warp roles (both passes): warps 0-7 consumers (split -> TMEM, epilogue; warp w
// owns TMEM lanes 32 (w % 4) of half w / 4), warps 8-11 producers (cp.async ring),
// warp 12 MMA issuer.  mbarriers only -- no CTA-wide barrier in the main loop.
constexpr int kWsThreads = 320;   // warps 0-7 consumers, warp 8 TMA producer, warp 9 MMA issuer
constexpr int kProducerWarp = 8;
constexpr int kMmaWarp = 9;

struct WsBars {
  uint64_t full[3];   // TMA -> consumers/MMA: stage landed (expect_tx)
  uint64_t xfree[3];  // consumers -> producer: raw stage read (count 256)
  uint64_t sfree[3];  // MMA -> producer: smem operand of the stage consumed (count 1)
  uint64_t tfull[2];  // consumers -> MMA: TMEM (and core) operand buffer b written (count 256)
  uint64_t tfree[2];  // MMA -> consumers: operand buffer b consumed (count 1)
  uint64_t accdone;   // MMA -> consumers: accumulators final (count 1)
};

__device__ __forceinline__ void ws_init(WsBars* b) {
  for (int i = 0; i < 3; ++i) {
    mbar_init(&b->full[i], 1);
    mbar_init(&b->xfree[i], 256);
    mbar_init(&b->sfree[i], 1);
  }
  for (int i = 0; i < 2; ++i) {
    mbar_init(&b->tfull[i], 256);
    mbar_init(&b->tfree[i], 1);
  }
  mbar_init(&b->accdone, 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
}

// Producer (one thread): wait until the slot's previous contents were consumed,
// arm the full barrier with the stage's bytes, issue the TMA loads.
template <typename IssueFn>
__device__ __forceinline__ void ws_produce(WsBars* bars, int nst, bool needs_sfree, uint32_t bytes, IssueFn issue) {
  constexpr int ST = 3;
  for (int s = 0; s < nst; ++s) {
    const int slot = s % ST;
    if (s >= ST) {
      const uint32_t ph = ((s / ST) - 1) & 1;
      mbar_wait(&bars->xfree[slot], ph);
      if (needs_sfree) mbar_wait(&bars->sfree[slot], ph);
    }
    mbar_expect_tx(&bars->full[slot], bytes);
    issue(s, slot, &bars->full[slot]);
  }
}

// ---------------------------------------------------------------------------
// A-pass: Aout[r][f] = alpha * sum_t X[r][t] S[f][t] for r < rows (<= 256).
// tmX: X-hat [rows_total][ldx] box {32, 256} SW128;  tmS: [2 np][ldx] (hi rows
// then lo rows) box {32, NP} SW128 -> directly the UMMA K-major SW128 layout.
// ---------------------------------------------------------------------------
template <int NP>
__global__ void __launch_bounds__(kWsThreads) k_tc_apass(const __grid_constant__ CUtensorMap tmX,
                                                          const __grid_constant__ CUtensorMap tmS, int np,
                                                          int ncontract, float* __restrict__ Aout, int64_t lda,
                                                          float alpha, const ItemA* __restrict__ items) {
  constexpr int ST = 3;
  constexpr int XB = 256 * kTcBK * 4;   // bytes per X tile
  constexpr int SB = NP * kTcBK * 4;    // bytes per S tile (hi or lo)
  constexpr int STAGE = XB + 2 * SB;
  extern __shared__ __align__(1024) uint8_t smem8[];
  uint8_t* smem = smem8 + ((1024 - (smem_u32(smem8) & 1023)) & 1023);
  __shared__ __align__(8) WsBars bars;
  __shared__ uint32_t tmem_base;
  const ItemA it = items[blockIdx.x];
  const int row0 = (int)(it.o_off / lda);   // global voxel row of the tile
  const int rows = it.rows;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nst = ncontract / kTcBK;

  if (warp == 0) tmem_alloc(&tmem_base, 512);
  if (tid == 0) ws_init(&bars);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == kProducerWarp) {
    if (lane == 0) {
      ws_produce(&bars, nst, true, (uint32_t)STAGE, [&](int s, int slot, uint64_t* bar) {
        uint8_t* st = smem + slot * STAGE;
        const int t0 = s * kTcBK;
        tma_load_2d(st, &tmX, t0, row0, bar);
        tma_load_2d(st + XB, &tmS, t0, 0, bar);
        tma_load_2d(st + XB + SB, &tmS, t0, np, bar);
      });
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(128, NP);
      for (int s = 0; s < nst; ++s) {
        const int b = s & 1, slot = s % ST;
        mbar_wait(&bars.tfull[b], (s >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t bh = smem_u32(smem + slot * STAGE + XB), bl = bh + SB;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t acc = tmem + 128u * hh;
          const uint32_t ar = tmem + abuf_col(b, hh), al = ar + 32;
#pragma unroll
          for (int ks = 0; ks < kTcBK / 8; ++ks) {
            const uint64_t dbh = umma_desc_sw128(bh + ks * 32);
            const uint64_t dbl = umma_desc_sw128(bl + ks * 32);
            mma_tf32_ts(acc, ar + ks * 8, dbh, idesc, (s | ks) != 0);
            mma_tf32_ts(acc, ar + ks * 8, dbl, idesc, 1);
            mma_tf32_ts(acc, al + ks * 8, dbh, idesc, 1);
          }
        }
        mma_commit(&bars.tfree[b]);
        mma_commit(&bars.sfree[slot]);
      }
      mma_commit(&bars.accdone);
    }
  } else {
    const int h = warp >> 2, q = warp & 3;
    const int row = 128 * h + 32 * q + lane;
    const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);
    for (int s = 0; s < nst; ++s) {
      const int b = s & 1, slot = s % ST;
      mbar_wait(&bars.full[slot], (s / ST) & 1);
      if (s >= 2) mbar_wait(&bars.tfree[b], ((s - 2) >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      // SW128 row: 16-byte chunk j of row r sits at chunk position j ^ (r & 7)
      const uint8_t* xr = smem + slot * STAGE + row * 128;
      float vals[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = *reinterpret_cast<const float4*>(xr + ((j ^ (row & 7)) << 4));
        vals[4 * j] = v.x;
        vals[4 * j + 1] = v.y;
        vals[4 * j + 2] = v.z;
        vals[4 * j + 3] = v.w;
      }
      mbar_arrive(&bars.xfree[slot]);
      store_split_row(tlane, abuf_col(b, h), vals);
      asm volatile("tcgen05.wait::st.sync.aligned;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&bars.tfull[b]);
    }
    mbar_wait(&bars.accdone, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    float* out = Aout + it.o_off;
#pragma unroll
    for (int c0 = 0; c0 < NP; c0 += 16) {
      float v[16];
      tmem_ld16(tlane + 128u * h + c0, v);
      if (row < rows) {
        float4* o = reinterpret_cast<float4*>(out + (int64_t)row * lda + c0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          o[j] = make_float4(alpha * v[4 * j], alpha * v[4 * j + 1], alpha * v[4 * j + 2], alpha * v[4 * j + 3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 512);
}

template <int NP>
cudaError_t run_apass(const CUtensorMap& tmX, const CUtensorMap& tmS, int np, int64_t ncontract, float* A,
                      int64_t lda, float alpha, const ItemA* items, int n_items, cudaStream_t st) {
  constexpr int bytes = 3 * (256 * kTcBK + 2 * NP * kTcBK) * 4 + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_tc_apass<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  k_tc_apass<NP><<<n_items, kWsThreads, bytes, st>>>(tmX, tmS, np, (int)ncontract, A, lda, alpha, items);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// B-pass: out[f][t0 + t] = sum_{v < rows} A[v][f] X[v][t0 + t] for t < 256, f < orows.
// tmXb: X-hat box {256, 32} (no swizzle); tmA: fp32 A [rows_total][np] box {NP, 32}.
// The X^T tile goes to TMEM (A operand); the A features tile is split +
// transposed into the K-major core layout in smem (B operand).  Voxel rows
// past the chunk are masked by the consumers (TMA loads whole boxes).
// ---------------------------------------------------------------------------
constexpr int kBT = 256;

template <int NP>
__global__ void __launch_bounds__(kWsThreads) k_tc_bpass(const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmXb, int64_t ldx,
                                                          double* __restrict__ out, int64_t ldo, int orows,
                                                          const ItemE* __restrict__ items) {
  constexpr int ST = 3;
  constexpr int XB = kTcBK * kBT * 4;   // raw X stage bytes
  constexpr int AB = kTcBK * NP * 4;    // raw A stage bytes
  constexpr int CT = NP * kTcBK;        // core tile floats (hi or lo)
  extern __shared__ __align__(1024) uint8_t smem8[];
  uint8_t* smem = smem8 + ((1024 - (smem_u32(smem8) & 1023)) & 1023);
  float* core = reinterpret_cast<float*>(smem);                  // [2 buffers][hi, lo]
  uint8_t* raw = smem + 2 * 2 * CT * 4;                          // [ST][rawX, rawA]
  __shared__ __align__(8) WsBars bars;
  __shared__ uint32_t tmem_base;
  const ItemE it = items[blockIdx.x];
  const int vrow0 = (int)(it.l_off / NP);          // first voxel row of the chunk (A row stride np == NP)
  const int t0 = (int)(it.r_off - (int64_t)vrow0 * ldx);
  const int rows = it.rows, ncols = it.ncols;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nst = (rows + kTcBK - 1) / kTcBK;

  if (warp == 0) tmem_alloc(&tmem_base, 512);
  if (tid == 0) ws_init(&bars);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == kProducerWarp) {
    if (lane == 0) {
      ws_produce(&bars, nst, false, (uint32_t)(XB + AB), [&](int s, int slot, uint64_t* bar) {
        uint8_t* rx = raw + slot * (XB + AB);
        tma_load_2d(rx, &tmXb, t0, vrow0 + s * kTcBK, bar);
        tma_load_2d(rx + XB, &tmA, 0, vrow0 + s * kTcBK, bar);
      });
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(128, NP);
      for (int s = 0; s < nst; ++s) {
        const int b = s & 1;
        mbar_wait(&bars.tfull[b], (s >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const float* ch = core + b * 2 * CT;
        const uint32_t bh = smem_u32(ch), bl = smem_u32(ch + CT);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t acc = tmem + 128u * hh;
          const uint32_t xr = tmem + abuf_col(b, hh), xl = xr + 32;
#pragma unroll
          for (int ks = 0; ks < kTcBK / 8; ++ks) {
            const uint64_t dbh = umma_desc(bh + ks * 256, 128, kTcBK * 32);
            const uint64_t dbl = umma_desc(bl + ks * 256, 128, kTcBK * 32);
            mma_tf32_ts(acc, xr + ks * 8, dbh, idesc, (s | ks) != 0);
            mma_tf32_ts(acc, xr + ks * 8, dbl, idesc, 1);
            mma_tf32_ts(acc, xl + ks * 8, dbh, idesc, 1);
          }
        }
        mma_commit(&bars.tfree[b]);
      }
      mma_commit(&bars.accdone);
    }
  } else {
    const int h = warp >> 2, q = warp & 3;
    const int tcol = 128 * h + 32 * q + lane;
    const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);
    for (int s = 0; s < nst; ++s) {
      const int b = s & 1, slot = s % ST;
      const int valid = min(kTcBK, rows - s * kTcBK);   // voxel rows of this stage inside the chunk
      mbar_wait(&bars.full[slot], (s / ST) & 1);
      if (s >= 2) mbar_wait(&bars.tfree[b], ((s - 2) >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const float* rx = reinterpret_cast<const float*>(raw + slot * (XB + AB));
      const float* ra = reinterpret_cast<const float*>(raw + slot * (XB + AB) + XB);
      float vals[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) vals[k] = k < valid ? rx[k * kBT + tcol] : 0.0f;
      float* ch = core + b * 2 * CT;
      float* cl = ch + CT;
      for (int e = tid; e < CT; e += 256) {
        const int r = (e >> 8) * 8 + ((e >> 2) & 7);   // feature
        const int k = ((e >> 5) & 7) * 4 + (e & 3);    // voxel in the stage
        const float a = k < valid ? ra[k * NP + r] : 0.0f;
        const float hi = tf32_hi(a);
        ch[e] = hi;
        cl[e] = a - hi;
      }
      mbar_arrive(&bars.xfree[slot]);
      store_split_row(tlane, abuf_col(b, h), vals);
      asm volatile("tcgen05.wait::st.sync.aligned;");
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(&bars.tfull[b]);
    }
    mbar_wait(&bars.accdone, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    double* ob = out + it.o_off;
#pragma unroll
    for (int c0 = 0; c0 < NP; c0 += 16) {
      float v[16];
      tmem_ld16(tlane + 128u * h + c0, v);
      if (tcol < ncols) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < orows) ob[(int64_t)(c0 + j) * ldo + tcol] = (double)v[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 512);
}

template <int NP>
cudaError_t run_bpass(const CUtensorMap& tmA, const CUtensorMap& tmXb, int64_t ldx, double* out, int64_t ldo,
                      int orows, const ItemE* items, int n_items, cudaStream_t st) {
  constexpr int bytes = (2 * 2 * NP * kTcBK + 3 * (kTcBK * kBT + kTcBK * NP)) * 4 + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_tc_bpass<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  k_tc_bpass<NP><<<n_items, kWsThreads, bytes, st>>>(tmA, tmXb, ldx, out, ldo, orows, items);
  return cudaGetLastError();
}

}  // namespace

int tc_np(int k) { return (k + 15) / 16 * 16; }

bool tc_supported(int k) { return k >= 1 && tc_np(k) <= 128; }

// ---------------------------------------------------------------------------
// tensor maps (host): cuTensorMapEncodeTiled through the runtime's driver entry point
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D fp32 map over [outer][inner] (row pitch in floats), box {box_inner, box_outer}
cudaError_t make_map_f32(TmaMap* m, const float* base, int64_t inner, int64_t outer, int64_t pitch,
                         int box_inner, int box_outer, bool swizzle128) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(m->opaque), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<float*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 3-D int8 map over int8 slice records Q[n][rows][lq] (bytes), box {128, box_rows, 1}, SWIZZLE_128B
cudaError_t make_map_q(TmaMap* m, const int8_t* base, int64_t lq, int64_t rows, int64_t n, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {(cuuint64_t)lq, (cuuint64_t)rows, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)lq, (cuuint64_t)(lq * rows)};
  cuuint32_t box[3] = {128, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(m->opaque), CU_TENSOR_MAP_DATA_TYPE_UINT8, 3,
                  const_cast<int8_t*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 4-D int8 map over row-slice records R[n][rows][ldx / 32][8 slots][32 B] with
// the dims ordered {32 B, row, slot index (k-block * 8 + slot), n}
// (non-monotonic strides) and box {32, 64, 8, 1}, SWIZZLE_32B: one load lands
// as [slot][row][32 B], so slots j and j + 1 of 64 rows form one 128-row
// K-major SW32 operand (the N = 128 slice pairs of the int8 row GEMMs)
cudaError_t make_map_q8(TmaMap* m, const int8_t* base, int64_t lq, int64_t rows, int64_t n, int slots) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[4] = {32, (cuuint64_t)rows, (cuuint64_t)(lq / 32), (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)lq, 32, (cuuint64_t)(lq * rows)};
  cuuint32_t box[4] = {32, 64, (cuuint32_t)slots, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(m->opaque), CU_TENSOR_MAP_DATA_TYPE_UINT8, 4,
                  const_cast<int8_t*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 5-D int8 map over the same records Q[n][ldx][nvb][8 slots][32 voxels] with the
// dims ordered {32 voxels, TR, voxel block, slot, subject} (non-monotonic
// strides) and box {32, 32, 4, 7, 1}, SWIZZLE_32B: one load lands as
// [slot][vb][t][32 B], per slot the MN-major operand of 128 voxels x 32 TRs
// (layout verified by tools/tma5d_probe.cu)
cudaError_t make_map_q5(TmaMap* m, const int8_t* base, int64_t lq, int64_t ldx, int64_t n, int nsl) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const int rec = oz_record_bytes(nsl);
  cuuint64_t dims[5] = {32, (cuuint64_t)ldx, (cuuint64_t)(lq / rec), (cuuint64_t)(rec / 32), (cuuint64_t)n};
  cuuint64_t strides[4] = {(cuuint64_t)lq, (cuuint64_t)rec, 32, (cuuint64_t)(lq * ldx)};
  cuuint32_t box[5] = {32, 32, 4, (cuuint32_t)nsl, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(m->opaque), CU_TENSOR_MAP_DATA_TYPE_UINT8, 5,
                  const_cast<int8_t*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_tc_apass(int np, const TmaMap& tmX, const TmaMap& tmS, int64_t ncontract, float* A, int64_t lda,
                            float alpha, const ItemA* items, int n_items, cudaStream_t st) {
  if (ncontract % kTcBK != 0) return cudaErrorInvalidValue;
  const CUtensorMap& mx = *reinterpret_cast<const CUtensorMap*>(tmX.opaque);
  const CUtensorMap& ms = *reinterpret_cast<const CUtensorMap*>(tmS.opaque);
  switch (np) {
#define CASE_TA(N) \
  case N: return run_apass<N>(mx, ms, np, ncontract, A, lda, alpha, items, n_items, st);
    CASE_TA(16) CASE_TA(32) CASE_TA(48) CASE_TA(64) CASE_TA(80) CASE_TA(96) CASE_TA(112) CASE_TA(128)
#undef CASE_TA
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace srm

namespace srm {

cudaError_t launch_tc_bpass(int np, const TmaMap& tmA, const TmaMap& tmXb, int64_t ldx, double* out, int64_t ldo,
                            int orows, const ItemE* items, int n_items, cudaStream_t st) {
  const CUtensorMap& ma = *reinterpret_cast<const CUtensorMap*>(tmA.opaque);
  const CUtensorMap& mx = *reinterpret_cast<const CUtensorMap*>(tmXb.opaque);
  switch (np) {
#define CASE_TB(N) \
  case N: return run_bpass<N>(ma, mx, ldx, out, ldo, orows, items, n_items, st);
    CASE_TB(16) CASE_TB(32) CASE_TB(48) CASE_TB(64) CASE_TB(80) CASE_TB(96) CASE_TB(112) CASE_TB(128)
#undef CASE_TB
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace srm
