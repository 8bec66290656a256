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
#include "common.cuh"
#include "kernels.h"

namespace srm {

namespace {

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

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(smem_u32(bar)), "r"(parity));
  }
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void tmem_free(uint32_t base, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
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

// ---------------------------------------------------------------------------
// A-pass: Aout[r][f] = alpha * sum_t X[r][t] S[f][t] for r < rows (<= 256)
// ---------------------------------------------------------------------------
template <int NP, int STAGES>
__global__ void __launch_bounds__(kTcT) k_tc_apass(const float* __restrict__ X, int64_t ldx,
                                                    const float* __restrict__ Shi, const float* __restrict__ Slo,
                                                    int64_t lds, int ncontract, float* __restrict__ Aout,
                                                    int64_t lda, float alpha, const ItemA* __restrict__ items) {
  constexpr int XS = 256 * kXStride;  // floats per raw X stage
  constexpr int SS = NP * kTcBK;      // floats per S tile (hi or lo)
  constexpr int STAGE = XS + 2 * SS;
  extern __shared__ __align__(1024) float smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const ItemA it = items[blockIdx.x];
  const float* Xb = X + it.x_off;
  const int rows = it.rows;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = warp >> 2, q = warp & 3;
  const int row = 128 * h + 32 * q + lane;
  const int nst = ncontract / kTcBK;

  if (warp == 0) tmem_alloc(&tmem_base, 512);
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);

  auto load = [&](int s) {
    float* xs = smem + (s % STAGES) * STAGE;
    float* sh = xs + XS;
    float* sl = sh + SS;
    const int t0 = s * kTcBK;
    for (int i = tid; i < 256 * 8; i += kTcT) {
      const int r = i >> 3, c = (i & 7) * 4;
      const bool ok = r < rows;
      cp_async16(xs + r * kXStride + c, Xb + (ok ? (int64_t)r * ldx + t0 + c : 0), ok);
    }
    for (int i = tid; i < NP * 8; i += kTcT) {
      // warp-contiguous core writes: 8 consecutive threads fill one 128-B core matrix
      const int core = i >> 3, rr = i & 7;
      const int r = (core >> 3) * 8 + rr, c = (core & 7) * 4;
      cp_async16(sh + kcore(r, c), Shi + (int64_t)r * lds + t0 + c, true);
      cp_async16(sl + kcore(r, c), Slo + (int64_t)r * lds + t0 + c, true);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nst) load(s);
    cp_async_commit();
  }
  constexpr uint32_t idesc = idesc_tf32(128, NP);
  for (int s = 0; s < nst; ++s) {
    const int b = s & 1;
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    // the TMEM A buffer b was read by the MMAs of stage s - 2
    if (s >= 2) mbar_wait(&mbar[b], ((s - 2) >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    {
      const float* xr = smem + (s % STAGES) * STAGE + row * kXStride;
      float vals[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 v = *reinterpret_cast<const float4*>(xr + 4 * j);
        vals[4 * j] = v.x;
        vals[4 * j + 1] = v.y;
        vals[4 * j + 2] = v.z;
        vals[4 * j + 3] = v.w;
      }
      store_split_row(tlane, abuf_col(b, h), vals);
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const float* sh = smem + (s % STAGES) * STAGE + XS;
      const uint32_t bh = smem_u32(sh), bl = smem_u32(sh + SS);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t acc = tmem + 128u * hh;
        const uint32_t ar = tmem + abuf_col(b, hh), al = ar + 32;
#pragma unroll
        for (int ks = 0; ks < kTcBK / 8; ++ks) {
          const uint64_t dbh = umma_desc(bh + ks * 256, 128, kTcBK * 32);
          const uint64_t dbl = umma_desc(bl + ks * 256, 128, kTcBK * 32);
          mma_tf32_ts(acc, ar + ks * 8, dbh, idesc, (s | ks) != 0);
          mma_tf32_ts(acc, ar + ks * 8, dbl, idesc, 1);
          mma_tf32_ts(acc, al + ks * 8, dbh, idesc, 1);
        }
      }
      mma_commit(&mbar[b]);
    }
    // refill the stage read by the MMAs of s - 1 (its S tile) with stage s + STAGES - 1
    const int ns = s + STAGES - 1;
    if (ns < nst) {
      if (s >= 1) mbar_wait(&mbar[(s - 1) & 1], ((s - 1) >> 1) & 1);
      load(ns);
    }
    cp_async_commit();
  }
  cp_async_wait<0>();
  mbar_wait(&mbar[(nst - 1) & 1], ((nst - 1) >> 1) & 1);
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
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 512);
}

template <int NP>
cudaError_t run_apass(const float* X, int64_t ldx, const float* Shi, const float* Slo, int64_t lds,
                      int64_t ncontract, float* A, int64_t lda, float alpha, const ItemA* items, int n_items,
                      cudaStream_t st) {
  constexpr int STAGES = 3;
  constexpr int bytes = STAGES * (256 * kXStride + 2 * NP * kTcBK) * 4;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_tc_apass<NP, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  k_tc_apass<NP, STAGES><<<n_items, kTcT, bytes, st>>>(X, ldx, Shi, Slo, lds, (int)ncontract, A, lda, alpha, items);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// B-pass: out[f][t0 + t] = sum_{v < rows} A[v][f] X[v][t0 + t] for t < 256, f < orows.
// X^T tile (t lanes x 32 v) goes to TMEM as the A operand; the A features tile
// is split + transposed into the K-major core layout in smem (B operand).
// ---------------------------------------------------------------------------
constexpr int kBT = 256;      // TRs per tile (two 128-lane halves)
constexpr int kAStr = 136;    // raw A stage row stride (floats): == 8 mod 32

template <int NP, int STAGES>
__global__ void __launch_bounds__(kTcT) k_tc_bpass(const float* __restrict__ A, int64_t lda,
                                                    const float* __restrict__ X, int64_t ldx,
                                                    double* __restrict__ out, int64_t ldo, int orows,
                                                    const ItemE* __restrict__ items) {
  constexpr int XR = kTcBK * kBT;     // raw X stage floats
  constexpr int AR = kTcBK * kAStr;   // raw A stage floats
  constexpr int CT = NP * kTcBK;      // core tile floats (hi or lo)
  extern __shared__ __align__(1024) float smem[];
  float* core = smem;                               // [2 buffers][hi, lo]
  float* raw = smem + 2 * 2 * CT;                   // [STAGES][rawX, rawA]
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const ItemE it = items[blockIdx.x];
  const float* Ab = A + it.l_off;
  const float* Xb = X + it.r_off;
  const int rows = it.rows, ncols = it.ncols;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = warp >> 2, q = warp & 3;
  const int tcol = 128 * h + 32 * q + lane;
  const int nst = (rows + kTcBK - 1) / kTcBK;

  if (warp == 0) tmem_alloc(&tmem_base, 512);
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);

  auto load = [&](int s) {
    float* rx = raw + (s % STAGES) * (XR + AR);
    float* ra = rx + XR;
    const int v0 = s * kTcBK;
    for (int i = tid; i < kTcBK * (kBT / 4); i += kTcT) {
      const int r = i >> 6, c = (i & 63) * 4;
      const bool ok = (v0 + r) < rows && c < ncols;
      cp_async16(rx + r * kBT + c, Xb + (ok ? (int64_t)(v0 + r) * ldx + c : 0), ok);
    }
    for (int i = tid; i < kTcBK * (NP / 4); i += kTcT) {
      const int r = i / (NP / 4), c = (i - r * (NP / 4)) * 4;
      const bool ok = (v0 + r) < rows;
      cp_async16(ra + r * kAStr + c, Ab + (ok ? (int64_t)(v0 + r) * lda + c : 0), ok);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nst) load(s);
    cp_async_commit();
  }
  constexpr uint32_t idesc = idesc_tf32(128, NP);
  for (int s = 0; s < nst; ++s) {
    const int b = s & 1;
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (s >= 2) mbar_wait(&mbar[b], ((s - 2) >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const float* rx = raw + (s % STAGES) * (XR + AR);
    const float* ra = rx + XR;
    {
      float vals[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) vals[k] = rx[k * kBT + tcol];
      store_split_row(tlane, abuf_col(b, h), vals);
    }
    float* ch = core + b * 2 * CT;
    float* cl = ch + CT;
    for (int e = tid; e < CT; e += kTcT) {
      const int r = (e >> 8) * 8 + ((e >> 2) & 7);   // feature
      const int k = ((e >> 5) & 7) * 4 + (e & 3);    // voxel in the stage
      const float a = ra[k * kAStr + r];
      const float hi = tf32_hi(a);
      ch[e] = hi;
      cl[e] = a - hi;
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t bh = smem_u32(ch), bl = smem_u32(cl);
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
      mma_commit(&mbar[b]);
    }
    if (s + STAGES - 1 < nst) load(s + STAGES - 1);  // raw stage (s-1) % STAGES was consumed above
    cp_async_commit();
  }
  cp_async_wait<0>();
  mbar_wait(&mbar[(nst - 1) & 1], ((nst - 1) >> 1) & 1);
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
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 512);
}

template <int NP>
cudaError_t run_bpass(const float* A, int64_t lda, const float* X, int64_t ldx, double* out, int64_t ldo,
                      int orows, const ItemE* items, int n_items, cudaStream_t st) {
  constexpr int STAGES = 3;
  constexpr int bytes = (2 * 2 * NP * kTcBK + STAGES * (kTcBK * kBT + kTcBK * kAStr)) * 4;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_tc_bpass<NP, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  k_tc_bpass<NP, STAGES><<<n_items, kTcT, bytes, st>>>(A, lda, X, ldx, out, ldo, orows, items);
  return cudaGetLastError();
}

}  // namespace

int tc_np(int k) { return (k + 15) / 16 * 16; }

bool tc_supported(int k) { return k >= 1 && tc_np(k) <= 128; }

cudaError_t launch_tc_apass(int np, const float* X, int64_t ldx, const float* Shi, const float* Slo, int64_t lds,
                            int64_t ncontract, float* A, int64_t lda, float alpha, const ItemA* items, int n_items,
                            cudaStream_t st) {
  if (ncontract % kTcBK != 0) return cudaErrorInvalidValue;
  switch (np) {
    case 16: return run_apass<16>(X, ldx, Shi, Slo, lds, ncontract, A, lda, alpha, items, n_items, st);
    case 32: return run_apass<32>(X, ldx, Shi, Slo, lds, ncontract, A, lda, alpha, items, n_items, st);
    case 48: return run_apass<48>(X, ldx, Shi, Slo, lds, ncontract, A, lda, alpha, items, n_items, st);
    case 64: return run_apass<64>(X, ldx, Shi, Slo, lds, ncontract, A, lda, alpha, items, n_items, st);
    case 80: return run_apass<80>(X, ldx, Shi, Slo, lds, ncontract, A, lda, alpha, items, n_items, st);
    case 96: return run_apass<96>(X, ldx, Shi, Slo, lds, ncontract, A, lda, alpha, items, n_items, st);
    case 112: return run_apass<112>(X, ldx, Shi, Slo, lds, ncontract, A, lda, alpha, items, n_items, st);
    case 128: return run_apass<128>(X, ldx, Shi, Slo, lds, ncontract, A, lda, alpha, items, n_items, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace srm

namespace srm {

cudaError_t launch_tc_bpass(int np, const float* A, int64_t lda, const float* X, int64_t ldx, double* out,
                            int64_t ldo, int orows, const ItemE* items, int n_items, cudaStream_t st) {
  switch (np) {
    case 16: return run_bpass<16>(A, lda, X, ldx, out, ldo, orows, items, n_items, st);
    case 32: return run_bpass<32>(A, lda, X, ldx, out, ldo, orows, items, n_items, st);
    case 48: return run_bpass<48>(A, lda, X, ldx, out, ldo, orows, items, n_items, st);
    case 64: return run_bpass<64>(A, lda, X, ldx, out, ldo, orows, items, n_items, st);
    case 80: return run_bpass<80>(A, lda, X, ldx, out, ldo, orows, items, n_items, st);
    case 96: return run_bpass<96>(A, lda, X, ldx, out, ldo, orows, items, n_items, st);
    case 112: return run_bpass<112>(A, lda, X, ldx, out, ldo, orows, items, n_items, st);
    case 128: return run_bpass<128>(A, lda, X, ldx, out, ldo, orows, items, n_items, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace srm
