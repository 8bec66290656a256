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

constexpr int kTcThreads = 128;
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

// ---------------------------------------------------------------------------
// A-pass: Aout[r][f] = alpha * sum_t X[r][t] (S_hi + S_lo)[f][t], r < rows (<= 128)
// ---------------------------------------------------------------------------
template <int NP, int STAGES>
__global__ void __launch_bounds__(kTcThreads) k_tc_apass(const float* __restrict__ X, int64_t ldx,
                                                          const float* __restrict__ Shi,
                                                          const float* __restrict__ Slo, int64_t lds,
                                                          int ncontract, float* __restrict__ Aout,
                                                          int64_t lda, float alpha,
                                                          const ItemA* __restrict__ items) {
  constexpr int XT = 128 * kTcBK;  // floats per X tile
  constexpr int ST = NP * kTcBK;   // floats per S tile
  constexpr int STAGE = 2 * XT + 2 * ST;
  extern __shared__ __align__(1024) float smem[];
  __shared__ __align__(8) uint64_t mbar[STAGES];
  __shared__ uint32_t tmem_base;
  const ItemA it = items[blockIdx.x];
  const float* Xb = X + it.x_off;
  const int rows = it.rows;
  const int tid = threadIdx.x;
  const int nst = ncontract / kTcBK;

  if (tid < 32) tmem_alloc(&tmem_base, tmem_cols(NP));
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  auto load = [&](int s) {
    float* base = smem + (s % STAGES) * STAGE;
    const int t0 = s * kTcBK;
    for (int i = tid; i < 128 * (kTcBK / 4); i += kTcThreads) {
      const int r = i >> 3, c = (i & 7) * 4;
      const bool ok = r < rows;
      cp_async16(base + kcore(r, c), Xb + (ok ? (int64_t)r * ldx + t0 + c : 0), ok);
    }
    float* sh = base + 2 * XT;
    float* sl = sh + ST;
    for (int i = tid; i < NP * (kTcBK / 4); i += kTcThreads) {
      const int r = i >> 3, c = (i & 7) * 4;
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
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    float* base = smem + (s % STAGES) * STAGE;
    float* xh = base;
    float* xl = base + XT;
    for (int e = tid; e < XT; e += kTcThreads) {
      const float x = xh[e];
      const float h = tf32_hi(x);
      xh[e] = h;
      xl[e] = x - h;
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_h = smem_u32(xh), a_l = smem_u32(xl);
      const uint32_t b_h = smem_u32(base + 2 * XT), b_l = smem_u32(base + 2 * XT + ST);
#pragma unroll
      for (int ks = 0; ks < kTcBK / 8; ++ks) {
        const uint32_t off = ks * 256;
        const uint64_t dah = umma_desc(a_h + off, 128, kTcBK * 32);
        const uint64_t dal = umma_desc(a_l + off, 128, kTcBK * 32);
        const uint64_t dbh = umma_desc(b_h + off, 128, kTcBK * 32);
        const uint64_t dbl = umma_desc(b_l + off, 128, kTcBK * 32);
        mma_tf32(tmem, dah, dbh, idesc, (s | ks) != 0);
        mma_tf32(tmem, dah, dbl, idesc, 1);
        mma_tf32(tmem, dal, dbh, idesc, 1);
      }
      mma_commit(&mbar[s % STAGES]);
    }
    const int ns = s + STAGES - 1;
    if (ns < nst) {
      if (s >= 1) mbar_wait(&mbar[(s - 1) % STAGES], ((s - 1) / STAGES) & 1);
      load(ns);
    }
    cp_async_commit();
  }
  cp_async_wait<0>();
  mbar_wait(&mbar[(nst - 1) % STAGES], ((nst - 1) / STAGES) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");

  const int warp = tid >> 5, lane = tid & 31;
  const int row = warp * 32 + lane;
  float* out = Aout + it.o_off;
#pragma unroll
  for (int c0 = 0; c0 < NP; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    if (row < rows) {
      float4* o = reinterpret_cast<float4*>(out + (int64_t)row * lda + c0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        o[j] = make_float4(alpha * v[4 * j], alpha * v[4 * j + 1], alpha * v[4 * j + 2], alpha * v[4 * j + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) tmem_free(tmem, tmem_cols(NP));
}

template <int NP>
cudaError_t run_apass(const float* X, int64_t ldx, const float* Shi, const float* Slo, int64_t lds,
                      int64_t ncontract, float* A, int64_t lda, float alpha, const ItemA* items, int n_items,
                      cudaStream_t st) {
  constexpr int STAGES = 3;
  constexpr int bytes = STAGES * (2 * 128 * kTcBK + 2 * NP * kTcBK) * 4;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_tc_apass<NP, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  k_tc_apass<NP, STAGES><<<n_items, kTcThreads, bytes, st>>>(X, ldx, Shi, Slo, lds, (int)ncontract, A, lda, alpha,
                                                            items);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// B-pass: out[f][t0 + t] = sum_{v < rows} A[v][f] X[v][t0 + t]  (f < 128, t < 128),
// written in fp64 for the fixed-order chunk reduction.  Raw tiles land
// row-major (padded) via cp.async; the split writes hi/lo transposed into the
// K-major core layout (contraction index v contiguous inside a core).
// ---------------------------------------------------------------------------
constexpr int kBN = 128;            // TRs per tile (MMA N)
constexpr int kBM = 128;            // features per tile (MMA M, zero-padded)
constexpr int kRawS = kBN + 8;      // raw row stride (floats), == 8 mod 32

__global__ void __launch_bounds__(kTcThreads) k_tc_bpass(const float* __restrict__ A, int64_t lda, int np,
                                                          const float* __restrict__ X, int64_t ldx,
                                                          double* __restrict__ out, int64_t ldo, int orows,
                                                          const ItemE* __restrict__ items) {
  constexpr int RAWX = kTcBK * kRawS;
  constexpr int RAWA = kTcBK * kRawS;
  constexpr int CT = kBN * kTcBK;  // floats per core tile (X or A)
  extern __shared__ __align__(1024) float smem[];
  float* hl = smem;                         // [2 buffers][xh, xl, ah, al] each CT floats
  float* raw = smem + 2 * 4 * CT;           // [2 buffers][rawX, rawA]
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const ItemE it = items[blockIdx.x];
  const float* Ab = A + it.l_off;
  const float* Xb = X + it.r_off;
  const int rows = it.rows, ncols = it.ncols;
  const int tid = threadIdx.x;
  const int nst = (rows + kTcBK - 1) / kTcBK;

  if (tid < 32) tmem_alloc(&tmem_base, kBN);
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  auto load = [&](int s) {
    float* rx = raw + (s & 1) * (RAWX + RAWA);
    float* ra = rx + RAWX;
    const int v0 = s * kTcBK;
    for (int i = tid; i < kTcBK * (kBN / 4); i += kTcThreads) {
      const int r = i >> 5, c = (i & 31) * 4;
      const bool okr = (v0 + r) < rows;
      const bool okx = okr && c < ncols;
      cp_async16(rx + r * kRawS + c, Xb + (okx ? (int64_t)(v0 + r) * ldx + c : 0), okx);
      const bool oka = okr && c < np;
      cp_async16(ra + r * kRawS + c, Ab + (oka ? (int64_t)(v0 + r) * lda + c : 0), oka);
    }
  };

  load(0);
  cp_async_commit();
  if (nst > 1) load(1);
  cp_async_commit();
  constexpr uint32_t idesc = idesc_tf32(kBM, kBN);
  for (int s = 0; s < nst; ++s) {
    cp_async_wait<1>();
    __syncthreads();
    // the hi/lo buffer of stage s was last read by the MMAs of stage s - 2
    if (s >= 2) mbar_wait(&mbar[s & 1], ((s - 2) >> 1) & 1);
    float* xh = hl + (s & 1) * 4 * CT;
    float* xl = xh + CT;
    float* ah = xl + CT;
    float* al = ah + CT;
    const float* rx = raw + (s & 1) * (RAWX + RAWA);
    const float* ra = rx + RAWX;
    for (int e = tid; e < CT; e += kTcThreads) {
      // core-major order: e = group*256 + kgroup*32 + (row & 7)*4 + (k & 3)
      const int row = (e >> 8) * 8 + ((e >> 2) & 7);
      const int k = ((e >> 5) & 7) * 4 + (e & 3);
      const float x = rx[k * kRawS + row];
      const float a = ra[k * kRawS + row];
      const float xhv = tf32_hi(x), ahv = tf32_hi(a);
      xh[e] = xhv;
      xl[e] = x - xhv;
      ah[e] = ahv;
      al[e] = a - ahv;
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int ks = 0; ks < kTcBK / 8; ++ks) {
        const uint32_t off = ks * 256;
        const uint64_t dah = umma_desc(smem_u32(ah) + off, 128, kTcBK * 32);
        const uint64_t dal = umma_desc(smem_u32(al) + off, 128, kTcBK * 32);
        const uint64_t dxh = umma_desc(smem_u32(xh) + off, 128, kTcBK * 32);
        const uint64_t dxl = umma_desc(smem_u32(xl) + off, 128, kTcBK * 32);
        mma_tf32(tmem, dah, dxh, idesc, (s | ks) != 0);
        mma_tf32(tmem, dah, dxl, idesc, 1);
        mma_tf32(tmem, dal, dxh, idesc, 1);
      }
      mma_commit(&mbar[s & 1]);
    }
    if (s + 2 < nst) load(s + 2);
    cp_async_commit();
  }
  cp_async_wait<0>();
  mbar_wait(&mbar[(nst - 1) & 1], ((nst - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid >> 5, lane = tid & 31;
  const int f = warp * 32 + lane;
  double* ob = out + it.o_off;
#pragma unroll
  for (int c0 = 0; c0 < kBN; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
    if (f < orows) {
#pragma unroll
      for (int j = 0; j < 16; j += 2)
        if (c0 + j < ncols)
          *reinterpret_cast<double2*>(ob + (int64_t)f * ldo + c0 + j) = make_double2((double)v[j], (double)v[j + 1]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) tmem_free(tmem, kBN);
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

cudaError_t launch_tc_bpass(const float* A, int64_t lda, int np, const float* X, int64_t ldx, double* out,
                            int64_t ldo, int orows, const ItemE* items, int n_items, cudaStream_t st) {
  constexpr int bytes = (2 * 4 * kBN * kTcBK + 2 * 2 * kTcBK * kRawS) * 4;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_tc_bpass, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  k_tc_bpass<<<n_items, kTcThreads, bytes, st>>>(A, lda, np, X, ldx, out, ldo, orows, items);
  return cudaGetLastError();
}

}  // namespace srm
