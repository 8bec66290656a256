// Streaming tall-skinny contractions of the SRM EM path on FP64 tensor cores.
//
//   contract_e ("V-contraction"):  out[m][n] = alpha * sum_v L[v][m] R[v][n]
//       E-step term  W_i^T Xhat_i          (srm.py:118, srm.py:151)
//       B_i = A_i^T Xhat_i, A_i^T A_i      (srm.py:147-151 via W = A M)
//       split over V chunks; each CTA writes one partial tile, reduced later
//       in a fixed order (deterministic, no atomics).
//   contract_a ("T-contraction"):  out[r][f] = alpha * sum_t X[r][t] S[f][t]
//       A_i = Xhat_i S^T / 2               (srm.py:147)
//
// Both kernels stage operand tiles through shared memory with a multi-stage
// cp.async (LDGSTS) pipeline and issue mma.sync.m8n8k4.f64 (SASS DMMA).  The
// smem row strides are padded so every fragment load of a half-warp hits 16
// distinct 8-byte bank pairs (stride == 4 mod 16 doubles).  X-hat may be
// fp32 in HBM (half the bytes); it is widened to fp64 on the fragment load,
// so all arithmetic is fp64 like the reference (kernels.py:40 upcasts).
#include "common.cuh"
#include "kernels.h"

namespace srm {

namespace {

constexpr int kThreads = 256;
constexpr int kTileN = 128;  // contract_e: output columns per CTA (8 warps x 16)
constexpr int kTileR = 128;  // contract_a: output rows per CTA (8 warps x 16)
constexpr int kBC = 16;      // contraction depth per pipeline stage
constexpr int kSmemBudget = 104 * 1024;

__host__ __device__ constexpr int pad4mod16(int n) { return n + ((4 - n) % 16 + 16) % 16; }

// apply_rows: rows of A staged per round (128, or 64 above kp = 112 where M
// and 128 rows of fp64 A would exceed shared memory)
__host__ __device__ constexpr int apply_rows_tile(int kp) { return kp > 112 ? 64 : 128; }

template <typename T>
__host__ __device__ constexpr int e_r_stride() { return sizeof(T) == 8 ? kTileN + 4 : kTileN + 8; }

// L-tile row stride: doubles == 4 mod 16, floats == 8 mod 32 (conflict-free fragments)
template <int KP, typename TL>
__host__ __device__ constexpr int e_l_stride() {
  return sizeof(TL) == 8 ? pad4mod16(KP) : KP + ((8 - KP) % 32 + 32) % 32;
}

template <int KP, typename TL, typename TR>
constexpr int e_stage_bytes() {
  return kBC * (e_l_stride<KP, TL>() * (int)sizeof(TL) + e_r_stride<TR>() * (int)sizeof(TR));
}

template <int KP, typename TL, typename TR>
constexpr int e_stages() {
  return (kSmemBudget / e_stage_bytes<KP, TL, TR>()) >= 4 ? 4
         : (kSmemBudget / e_stage_bytes<KP, TL, TR>()) >= 3 ? 3 : 2;
}

constexpr int kAStride = 20;  // == 4 mod 16 doubles; conflict-free for floats too

template <int KP, typename TX>
constexpr int a_stage_bytes() {
  return kTileR * kAStride * (int)sizeof(TX) + KP * kAStride * 8;
}

template <int KP, typename TX>
constexpr int a_stages() {
  return (kSmemBudget / a_stage_bytes<KP, TX>()) >= 4 ? 4
         : (kSmemBudget / a_stage_bytes<KP, TX>()) >= 3 ? 3 : 2;
}

__device__ __forceinline__ void store2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// ---------------------------------------------------------------------------
// V-contraction
// ---------------------------------------------------------------------------
template <int KP, typename TL, typename TR, int STAGES>
__global__ void __launch_bounds__(kThreads) k_contract_e(const TL* __restrict__ L, int64_t ldl,
                                                         const TR* __restrict__ R, int64_t ldr,
                                                         double* __restrict__ out, int64_t ldo,
                                                         double alpha,
                                                         const ItemE* __restrict__ items) {
  constexpr int SL = e_l_stride<KP, TL>();
  constexpr int SR = e_r_stride<TR>();
  constexpr int MT = KP / 8;
  constexpr int EPC = 16 / (int)sizeof(TR);  // elements per 16-byte chunk
  constexpr int LEPC = 16 / (int)sizeof(TL);
  constexpr int LCH = KP / LEPC;             // 16-byte chunks per L row
  constexpr int RCH = kTileN / EPC;          // 16-byte chunks per R row

  extern __shared__ __align__(16) unsigned char smem_raw[];
  TL* Ls = reinterpret_cast<TL*>(smem_raw);
  TR* Rs = reinterpret_cast<TR*>(smem_raw + STAGES * kBC * SL * (int)sizeof(TL));

  const ItemE it = items[blockIdx.x];
  const TL* Lb = L + it.l_off;
  const TR* Rb = R + it.r_off;
  const int rows = it.rows;
  const int ncols = it.ncols;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int nstages = (rows + kBC - 1) / kBC;

  auto load_stage = [&](int s, int buf) {
    const int r0 = s * kBC;
    TL* ld = Ls + buf * kBC * SL;
    for (int i = tid; i < kBC * LCH; i += kThreads) {
      const int r = i / LCH, c = (i - r * LCH) * LEPC;
      const bool ok = (r0 + r) < rows;
      cp_async16(ld + r * SL + c, Lb + (int64_t)(ok ? r0 + r : 0) * ldl + c, ok);
    }
    TR* rd = Rs + buf * kBC * SR;
    for (int i = tid; i < kBC * RCH; i += kThreads) {
      const int r = i / RCH, c = (i - r * RCH) * EPC;
      const bool ok = (r0 + r) < rows && c < ncols;
      cp_async16(rd + r * SR + c, Rb + (ok ? (int64_t)(r0 + r) * ldr + c : 0), ok);
    }
  };

  double acc[MT][2][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < 2; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nstages) load_stage(s, s);
    cp_async_commit();
  }

  const int ncol = warp * 16 + (lane >> 2);
  const int krow = lane & 3;
  for (int s = 0; s < nstages; ++s) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int ns = s + STAGES - 1;
      if (ns < nstages) load_stage(ns, ns % STAGES);
      cp_async_commit();
    }
    const int buf = s % STAGES;
    const TL* Lt = Ls + buf * kBC * SL;
    const TR* Rt = Rs + buf * kBC * SR;
#pragma unroll
    for (int kk = 0; kk < kBC; kk += 4) {
      const int cr = kk + krow;
      const double b0 = to_f64(Rt[cr * SR + ncol]);
      const double b1 = to_f64(Rt[cr * SR + ncol + 8]);
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const double a = to_f64(Lt[cr * SL + m * 8 + (lane >> 2)]);
        dmma(acc[m][0][0], acc[m][0][1], a, b0);
        dmma(acc[m][1][0], acc[m][1][1], a, b1);
      }
    }
  }
  cp_async_wait<0>();

  double* ob = out + it.o_off;
  const int mrows = it.mrows;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    const int row = m * 8 + (lane >> 2);
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      const int col = warp * 16 + n * 8 + 2 * (lane & 3);
      if (col < ncols && row < mrows) store2(ob + (int64_t)row * ldo + col, alpha * acc[m][n][0], alpha * acc[m][n][1]);
    }
  }
}

// ---------------------------------------------------------------------------
// T-contraction
// ---------------------------------------------------------------------------
template <int KP, typename TX, int STAGES>
__global__ void __launch_bounds__(kThreads) k_contract_a(const TX* __restrict__ X, int64_t ldx,
                                                         const double* __restrict__ S, int64_t lds,
                                                         int ncontract, double* __restrict__ out,
                                                         int64_t ldo, double alpha,
                                                         const ItemA* __restrict__ items) {
  constexpr int SX = kAStride;
  constexpr int SS = kAStride;
  constexpr int NT = KP / 8;
  constexpr int EPC = 16 / (int)sizeof(TX);
  constexpr int XCH = kBC / EPC;  // chunks per X row per stage
  constexpr int SCH = kBC / 2;    // chunks per S row per stage

  extern __shared__ __align__(16) unsigned char smem_raw[];
  TX* Xs = reinterpret_cast<TX*>(smem_raw);
  double* Ss = reinterpret_cast<double*>(smem_raw + STAGES * kTileR * SX * (int)sizeof(TX));

  const ItemA it = items[blockIdx.x];
  const TX* Xb = X + it.x_off;
  const int rows = it.rows;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int nstages = ncontract / kBC;

  auto load_stage = [&](int s, int buf) {
    const int t0 = s * kBC;
    TX* xd = Xs + buf * kTileR * SX;
    for (int i = tid; i < kTileR * XCH; i += kThreads) {
      const int r = i / XCH, c = (i - r * XCH) * EPC;
      const bool ok = r < rows;
      cp_async16(xd + r * SX + c, Xb + (ok ? (int64_t)r * ldx + t0 + c : 0), ok);
    }
    double* sd = Ss + buf * KP * SS;
    for (int i = tid; i < KP * SCH; i += kThreads) {
      const int r = i / SCH, c = (i - r * SCH) * 2;
      cp_async16(sd + r * SS + c, S + (int64_t)r * lds + t0 + c, true);
    }
  };

  double acc[2][NT][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nstages) load_stage(s, s);
    cp_async_commit();
  }

  const int arow = warp * 16 + (lane >> 2);
  const int kcol = lane & 3;
  for (int s = 0; s < nstages; ++s) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int ns = s + STAGES - 1;
      if (ns < nstages) load_stage(ns, ns % STAGES);
      cp_async_commit();
    }
    const int buf = s % STAGES;
    const TX* Xt = Xs + buf * kTileR * SX;
    const double* St = Ss + buf * KP * SS;
#pragma unroll
    for (int kk = 0; kk < kBC; kk += 4) {
      const double a0 = to_f64(Xt[arow * SX + kk + kcol]);
      const double a1 = to_f64(Xt[(arow + 8) * SX + kk + kcol]);
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const double b = St[(n * 8 + (lane >> 2)) * SS + kk + kcol];
        dmma(acc[0][n][0], acc[0][n][1], a0, b);
        dmma(acc[1][n][0], acc[1][n][1], a1, b);
      }
    }
  }
  cp_async_wait<0>();

  double* ob = out + it.o_off;
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    const int row = warp * 16 + m * 8 + (lane >> 2);
    if (row < rows) {
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int col = n * 8 + 2 * (lane & 3);
        store2(ob + (int64_t)row * ldo + col, alpha * acc[m][n][0], alpha * acc[m][n][1]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Gram tiles of X^T X (Gram path, one-time): out[m][n] = sum_v X[v][m0+m] X[v][n0+n]
// for 128 x 128 tiles.  4 x 2 warp grid (each warp 32 rows x 64 columns: 4 A and 8
// B fragments per 32 DMMA), 32-deep pipeline stages.  Diagonal tiles (item.pad
// = 1) skip the strictly-lower 64 x 64 block; the mirror kernel fills it.
// ---------------------------------------------------------------------------
constexpr int kGBC = 32;

template <typename TX>
__host__ __device__ constexpr int g_stride() { return sizeof(TX) == 8 ? 132 : 136; }

template <typename TX>
constexpr int g_stage_bytes() { return 2 * kGBC * g_stride<TX>() * (int)sizeof(TX); }

template <typename TX, int STAGES>
__global__ void __launch_bounds__(kThreads) k_gram128(const TX* __restrict__ X, int64_t ldx,
                                                      double* __restrict__ out, int64_t ldo,
                                                      const ItemE* __restrict__ items) {
  constexpr int SX = g_stride<TX>();
  constexpr int EPC = 16 / (int)sizeof(TX);
  constexpr int CH = 128 / EPC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TX* Ls = reinterpret_cast<TX*>(smem_raw);
  TX* Rs = Ls + STAGES * kGBC * SX;
  const ItemE it = items[blockIdx.x];
  const TX* Lb = X + it.l_off;
  const TX* Rb = X + it.r_off;
  const int rows = it.rows, ncols = it.ncols, mrows = it.mrows;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 1, wn = warp & 1;  // rows [32 wm, +32), cols [64 wn, +64)
  const bool skip = it.pad && (wm >= 2 * wn + 2);
  const int nstages = (rows + kGBC - 1) / kGBC;

  auto load_stage = [&](int s, int buf) {
    const int r0 = s * kGBC;
    TX* ld = Ls + buf * kGBC * SX;
    TX* rd = Rs + buf * kGBC * SX;
    for (int i = tid; i < kGBC * CH; i += kThreads) {
      const int r = i / CH, c = (i - r * CH) * EPC;
      const bool okr = (r0 + r) < rows;
      const bool okl = okr && c < mrows;
      const bool okc = okr && c < ncols;
      cp_async16(ld + r * SX + c, Lb + (okl ? (int64_t)(r0 + r) * ldx + c : 0), okl);
      cp_async16(rd + r * SX + c, Rb + (okc ? (int64_t)(r0 + r) * ldx + c : 0), okc);
    }
  };

  double acc[4][8][2];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int n = 0; n < 8; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nstages) load_stage(s, s);
    cp_async_commit();
  }
  const int arow = wm * 32 + (lane >> 2);
  const int bcol = wn * 64 + (lane >> 2);
  const int kr = lane & 3;
  for (int s = 0; s < nstages; ++s) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int ns = s + STAGES - 1;
      if (ns < nstages) load_stage(ns, ns % STAGES);
      cp_async_commit();
    }
    if (skip) continue;
    const TX* Lt = Ls + (s % STAGES) * kGBC * SX;
    const TX* Rt = Rs + (s % STAGES) * kGBC * SX;
#pragma unroll
    for (int kk = 0; kk < kGBC; kk += 4) {
      const int cr = (kk + kr) * SX;
      double a[4], b[8];
#pragma unroll
      for (int m = 0; m < 4; ++m) a[m] = to_f64(Lt[cr + arow + m * 8]);
#pragma unroll
      for (int n = 0; n < 8; ++n) b[n] = to_f64(Rt[cr + bcol + n * 8]);
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 8; ++n) dmma(acc[m][n][0], acc[m][n][1], a[m], b[n]);
    }
  }
  cp_async_wait<0>();
  if (skip) return;
  double* ob = out + it.o_off;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int row = wm * 32 + m * 8 + (lane >> 2);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int col = wn * 64 + n * 8 + 2 * (lane & 3);
      if (row < mrows && col < ncols) store2(ob + (int64_t)row * ldo + col, acc[m][n][0], acc[m][n][1]);
    }
  }
}

template <typename TX>
cudaError_t run_g(const TX* X, int64_t ldx, double* out, int64_t ldo, const ItemE* items, int n_items,
                  cudaStream_t stream) {
  constexpr int ST = 3;
  constexpr int bytes = ST * g_stage_bytes<TX>();
  auto kern = k_gram128<TX, ST>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  kern<<<n_items, kThreads, bytes, stream>>>(X, ldx, out, ldo, items);
  return cudaGetLastError();
}

template <int KP, typename TL, typename TR>
cudaError_t run_e(const TL* L, int64_t ldl, const TR* R, int64_t ldr, double* out, int64_t ldo,
                  double alpha, const ItemE* items, int n_items, cudaStream_t stream) {
  constexpr int ST = e_stages<KP, TL, TR>();
  constexpr int bytes = ST * e_stage_bytes<KP, TL, TR>();
  auto kern = k_contract_e<KP, TL, TR, ST>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  kern<<<n_items, kThreads, bytes, stream>>>(L, ldl, R, ldr, out, ldo, alpha, items);
  return cudaGetLastError();
}

template <int KP, typename TX>
cudaError_t run_a(const TX* X, int64_t ldx, const double* S, int64_t lds, int64_t ncontract,
                  double* out, int64_t ldo, double alpha, const ItemA* items, int n_items,
                  cudaStream_t stream) {
  constexpr int ST = a_stages<KP, TX>();
  constexpr int bytes = ST * a_stage_bytes<KP, TX>();
  auto kern = k_contract_a<KP, TX, ST>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  kern<<<n_items, kThreads, bytes, stream>>>(X, ldx, S, lds, (int)ncontract, out, ldo, alpha, items);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// W = A M on DMMA (srm.py:315-327 model.W via kernels.py:212 U V^T = A M):
// W[row0 + r][f] = sum_c A[row0 + r][c] M_i[c][f] for r < rows (<= 256), f < K.
// ---------------------------------------------------------------------------
template <int KP, typename TA>
__global__ void __launch_bounds__(kThreads) k_apply_rows(const TA* __restrict__ A, int64_t lda,
                                                         const double* __restrict__ Mall, int64_t mstride,
                                                         double* __restrict__ W, int K,
                                                         const ItemA* __restrict__ items) {
  constexpr int SA = pad4mod16(KP) + (sizeof(TA) == 4 ? 4 : 0);  // floats: == 8 mod 32 words
  constexpr int SM = pad4mod16(KP);
  constexpr int NT = KP / 8;
  constexpr int RT = apply_rows_tile(KP);  // rows staged per round: M and the row tile fit in shared memory
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Ms = reinterpret_cast<double*>(smem_raw);
  TA* As = reinterpret_cast<TA*>(smem_raw + KP * SM * 8);
  const ItemA it = items[blockIdx.x];
  const double* Mg = Mall + (int64_t)it.pad * mstride;
  const int64_t row0 = it.o_off / lda;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < KP * KP; e += kThreads) Ms[(e / KP) * SM + e % KP] = Mg[e];
  for (int half = 0; half * RT < it.rows; ++half) {
    const int r0 = half * RT;
    const int nr = min(RT, it.rows - r0);
    __syncthreads();
    for (int e = tid; e < RT * KP; e += kThreads) {
      const int r = e / KP, c = e - r * KP;
      As[r * SA + c] = r < nr ? A[(row0 + r0 + r) * lda + c] : TA(0);
    }
    __syncthreads();
    if (warp * 16 >= RT) continue;  // RT = 64: warps 4-7 only stage
    double acc[2][NT][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    const int arow = warp * 16 + (lane >> 2);
#pragma unroll 2
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const int kc = k0 + (lane & 3);
      const double a0 = to_f64(As[arow * SA + kc]);
      const double a1 = to_f64(As[(arow + 8) * SA + kc]);
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const double b = Ms[kc * SM + n * 8 + (lane >> 2)];
        dmma(acc[0][n][0], acc[0][n][1], a0, b);
        dmma(acc[1][n][0], acc[1][n][1], a1, b);
      }
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int r = warp * 16 + m * 8 + (lane >> 2);
      if (r < nr) {
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int f = n * 8 + 2 * (lane & 3);
          double* w = W + (row0 + r0 + r) * K;
          if (f < K) w[f] = acc[m][n][0];
          if (f + 1 < K) w[f + 1] = acc[m][n][1];
        }
      }
    }
  }
}

template <int KP, typename TA>
cudaError_t run_apply(const TA* A, int64_t lda, const double* M, int64_t mstride, double* W, int K,
                      const ItemA* items, int n_items, cudaStream_t st) {
  constexpr int SA = pad4mod16(KP) + (sizeof(TA) == 4 ? 4 : 0);
  constexpr int bytes = KP * pad4mod16(KP) * 8 + apply_rows_tile(KP) * SA * (int)sizeof(TA);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_apply_rows<KP, TA>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (n_items == 0) return cudaSuccess;
  k_apply_rows<KP, TA><<<n_items, kThreads, bytes, st>>>(A, lda, M, mstride, W, K, items);
  return cudaGetLastError();
}

}  // namespace

bool contract_kp_supported(int kp) { return kp >= 8 && kp <= 128 && kp % 8 == 0; }

cudaError_t launch_gram_tiles(int x_dtype, const void* X, int64_t ldx, double* out, int64_t ldo,
                              const ItemE* items, int n_items, cudaStream_t stream) {
  if (x_dtype == SRM_F64)
    return run_g<double>(static_cast<const double*>(X), ldx, out, ldo, items, n_items, stream);
  return run_g<float>(static_cast<const float*>(X), ldx, out, ldo, items, n_items, stream);
}

#define SRM_KP_CASES(F) \
  F(8) F(16) F(24) F(32) F(40) F(48) F(56) F(64) F(72) F(80) F(88) F(96) F(104) F(112) F(120) F(128)

cudaError_t launch_contract_e(int kp, int l_dtype, int r_dtype, const void* L, int64_t ldl, const void* R,
                              int64_t ldr, double* out, int64_t ldo, double alpha,
                              const ItemE* items, int n_items, cudaStream_t stream) {
  if (l_dtype == SRM_F32 && r_dtype == SRM_F64) return cudaErrorInvalidValue;
#define CASE_E(K)                                                                                  \
  case K:                                                                                          \
    if (l_dtype == SRM_F64 && r_dtype == SRM_F64)                                                  \
      return run_e<K, double, double>(static_cast<const double*>(L), ldl,                          \
                                      static_cast<const double*>(R), ldr, out, ldo, alpha, items,  \
                                      n_items, stream);                                            \
    if (l_dtype == SRM_F64)                                                                        \
      return run_e<K, double, float>(static_cast<const double*>(L), ldl,                           \
                                     static_cast<const float*>(R), ldr, out, ldo, alpha, items,    \
                                     n_items, stream);                                             \
    return run_e<K, float, float>(static_cast<const float*>(L), ldl, static_cast<const float*>(R), \
                                  ldr, out, ldo, alpha, items, n_items, stream);
  switch (kp) {
    SRM_KP_CASES(CASE_E)
    default:
      return cudaErrorInvalidValue;
  }
#undef CASE_E
}

cudaError_t launch_apply_rows(int kp, int a_dtype, const void* A, int64_t lda, const double* M, int64_t mstride,
                              double* W, int K, const ItemA* items, int n_items, cudaStream_t stream) {
#define CASE_W(KK)                                                                                   \
  case KK:                                                                                           \
    return a_dtype == SRM_F64                                                                        \
               ? run_apply<KK, double>(static_cast<const double*>(A), lda, M, mstride, W, K, items, \
                                       n_items, stream)                                              \
               : run_apply<KK, float>(static_cast<const float*>(A), lda, M, mstride, W, K, items,   \
                                      n_items, stream);
  switch (kp) {
    SRM_KP_CASES(CASE_W)
    default:
      return cudaErrorInvalidValue;
  }
#undef CASE_W
}

cudaError_t launch_contract_a(int kp, int x_dtype, const void* X, int64_t ldx, const double* S,
                              int64_t lds, int64_t ncontract, double* out, int64_t ldo,
                              double alpha, const ItemA* items, int n_items, cudaStream_t stream) {
  if (ncontract % kBC != 0) return cudaErrorInvalidValue;
#define CASE_A(K)                                                                              \
  case K:                                                                                      \
    return x_dtype == SRM_F64                                                                  \
               ? run_a<K, double>(static_cast<const double*>(X), ldx, S, lds, ncontract, out,  \
                                  ldo, alpha, items, n_items, stream)                          \
               : run_a<K, float>(static_cast<const float*>(X), ldx, S, lds, ncontract, out,    \
                                 ldo, alpha, items, n_items, stream);
  switch (kp) {
    SRM_KP_CASES(CASE_A)
    default:
      return cudaErrorInvalidValue;
  }
#undef CASE_A
}

}  // namespace srm
