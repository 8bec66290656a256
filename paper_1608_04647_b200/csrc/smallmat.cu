// K x K and per-subject kernels of the SRM EM path (sm_100a, fp64).
//
//   prep            srm.py:94-98 demean, kernels.py:45 finite check, and the
//                   loop-invariant trace_ata(Xhat) of srm.py:152 (hoisted)
//   reduce_chunks   fixed-order sum of the V-chunk partials of contract_e
//   eig_polar       kernels.py:190-212 polar factor through the K x K Gram:
//                   parallel cyclic Jacobi (round-robin pairs), warm-started
//                   from the previous iteration's eigenvectors;
//                   M = Q diag(lambda^-1/2) Q^T so that W = A M
//   apply_m         W_new^T Xhat = M^T (A^T Xhat) (srm.py:151 and the next
//                   E-step term srm.py:118) + the cross term <., S>
//   finalize_rho    srm.py:152-155 noise update with the 1e-12 floor
//   reduce_terms    srm.py:193-213 ordered accumulation of rho^-2 W^T Xhat
//   tail            srm.py:121-142: two SPD inverses (kernels.py:168-187, by a
//                   symmetric sweep with the same pivots as Cholesky),
//                   S, Sigma_s update + trace, Woodbury log-likelihood,
//                   tolerance statistic (srm.py:275-287)
//   apply_w         W_i = A_i M_i (model.W)
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "plan.h"

namespace srm {

namespace {

constexpr int kSmallThreads = 256;
constexpr int kMaxK = 128;

__device__ __forceinline__ double* rec_ptr(const DevPlan& p, int slot) {
  return p.terms + (int64_t)slot * p.term_stride;
}

__device__ __forceinline__ bool failed(const DevPlan& p) { return p.status[0] != 0; }

// ---------------------------------------------------------------------------
// prep: one warp per voxel row
// ---------------------------------------------------------------------------
// One warp per voxel row, kPrepRows rows per CTA.  On the int8 Gram path
// (p.cmax) the pass also keeps the per-column maxima of the stored |Xhat|
// (the slice exponents, like rowsq a statistic of the demeaned data):
// shared-memory atomics, then one global atomic per column per CTA.
constexpr int kPrepRows = 32;

template <typename TIN, typename TOUT>
__global__ void __launch_bounds__(kSmallThreads) k_prep(DevPlan p, int local, const TIN* __restrict__ x,
                                                        int64_t ld) {
  extern __shared__ unsigned long long cmax_s[];  // [ldx] when p.cmax
  const int64_t* sj = p.subj + (int64_t)local * kSubjCols;
  const int64_t row0 = sj[SC_ROW_OFF];
  const int64_t V = sj[SC_V];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool track = p.cmax != nullptr;
  if (track) {
    for (int64_t t = threadIdx.x; t < p.ldx; t += blockDim.x) cmax_s[t] = 0ull;
    __syncthreads();
  }
  for (int rr = 0; rr < kPrepRows / 8; ++rr) {
    const int64_t row = (int64_t)blockIdx.x * kPrepRows + rr * 8 + warp;
    if (row >= V) break;
    const TIN* xr = x + row * ld;
    double s = 0.0;
    bool finite = true;
    for (int64_t t = lane; t < p.T; t += 32) {
      const double v = to_f64(xr[t]);
      finite &= isfinite(v);
      s += v;
    }
    s = warp_sum(s);
    const bool all_finite = __all_sync(0xffffffffu, finite);
    if (!all_finite && lane == 0) raise_status(p.status, SRM_ERR_INVALID_INPUT, (int)sj[SC_GLOBAL], -1);
    const double mean = s / (double)p.T;
    TOUT* out = static_cast<TOUT*>(p.xhat) + (row0 + row) * p.ldx;
    double sq = 0.0;
    for (int64_t t = lane; t < p.ldx; t += 32) {
      double v = 0.0;
      if (t < p.T) {
        v = to_f64(xr[t]) - mean;
        sq += v * v;
      }
      const TOUT stored = static_cast<TOUT>(v);
      out[t] = stored;
      if (track && t < p.T) {
        const double a = fabs(to_f64(stored));
        if (a > 0.0) atomicMax(cmax_s + t, (unsigned long long)__double_as_longlong(a));
      }
    }
    sq = warp_sum(sq);
    if (lane == 0) {
      p.mu[row0 + row] = mean;
      p.rowsq[row0 + row] = sq;
    }
  }
  if (track) {
    __syncthreads();
    for (int64_t t = threadIdx.x; t < p.ldx; t += blockDim.x)
      if (cmax_s[t]) atomicMax(p.cmax + (int64_t)local * p.ldx + t, cmax_s[t]);
  }
}

// per subject: sum of row sums of squares in a fixed order; fills record scalars
__global__ void __launch_bounds__(kSmallThreads) k_subject_sqnorm(DevPlan p) {
  __shared__ double scratch[32];
  const int i = blockIdx.x;
  const int64_t* sj = p.subj + (int64_t)i * kSubjCols;
  const int64_t row0 = sj[SC_ROW_OFF], V = sj[SC_V];
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < V; r += kSmallThreads) s += p.rowsq[row0 + r];
  s = block_sum<kSmallThreads>(s, scratch);
  if (threadIdx.x == 0) {
    double* rec = rec_ptr(p, (int)sj[SC_SLOT]) + p.kp * p.ldx;
    rec[RC_RHO2] = 1.0;
    rec[RC_V] = (double)V;
    rec[RC_SQNORM] = s;
  }
}

// ---------------------------------------------------------------------------
// reduce_chunks: bred[i] = sum_c part[chunk0 + c] (fixed order)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads) k_reduce_chunks(DevPlan p) {
  const int i = p.sub0 + blockIdx.y;
  const int64_t* sj = p.subj + (int64_t)i * kSubjCols;
  const int64_t c0 = sj[SC_CHUNK0], nc = sj[SC_NCHUNK];
  const int64_t n2 = p.kp * p.ldo / 2;  // double2 elements
  const int64_t e = (int64_t)blockIdx.x * kSmallThreads + threadIdx.x;
  if (e >= n2) return;
  const double2* src = reinterpret_cast<const double2*>(p.part + c0 * p.kp * p.ldo) + e;
  double2 acc = src[0];
  for (int64_t c = 1; c < nc; ++c) {
    const double2 v = src[c * n2];
    acc.x += v.x;
    acc.y += v.y;
  }
  reinterpret_cast<double2*>(p.bred + (int64_t)i * p.kp * p.ldo)[e] = acc;
}

// ---------------------------------------------------------------------------
// Jacobi eigensolver on a symmetric n x n matrix in shared memory.
//   C (n x ld) is diagonalised in place, Q (n x ld) accumulates rotations
//   (Q <- Q J).  Round-robin ordering: n'/2 disjoint (p,q) planes per round,
//   n'-1 rounds per sweep; a sweep with no rotation ends the iteration.
// ---------------------------------------------------------------------------
struct JacobiScratch {
  double* cs;
  double* sn;
  int* pp;
  int* qq;
  int* rot;
};

__device__ int rr_slot(int i, int r, int np2) { return i == 0 ? 0 : 1 + ((i - 1 + r) % (np2 - 1)); }

// Returns the number of sweeps run.  Convergence: the off-diagonal Frobenius
// norm is at most 1e-15 of the matrix norm at the start of a sweep (eigen-
// value errors ~1e-15 |C|).  A purely relative per-entry test can stall on
// roundoff-level entries next to small eigenvalues; rotations on entries
// below 1e-18 |C| are skipped as noise.
__device__ int jacobi_eig(double* C, double* Q, int n, int ld, JacobiScratch js, int max_sweeps) {
  __shared__ double red_scratch[32];
  const int tid = threadIdx.x;
  const int np2 = (n + 1) & ~1;
  const int npairs = np2 / 2;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int a = e / n, b = e - a * n;
      const double v = C[a * ld + b];
      tot += v * v;
      if (a != b) off += v * v;
    }
    off = block_sum<kSmallThreads>(off, red_scratch);
    tot = block_sum<kSmallThreads>(tot, red_scratch);
    if (!(off > 1e-30 * tot)) break;  // also stops on NaN
    const double noise = 1e-18 * sqrt(tot);
    for (int r = 0; r < np2 - 1; ++r) {
      for (int j = tid; j < npairs; j += blockDim.x) {
        const int a = rr_slot(j, r, np2), b = rr_slot(np2 - 1 - j, r, np2);
        const int pi = min(a, b), qi = max(a, b);
        double c = 1.0, s = 0.0;
        if (qi < n) {
          const double apq = C[pi * ld + qi];
          const double app = C[pi * ld + pi];
          const double aqq = C[qi * ld + qi];
          if (fabs(apq) > noise && fabs(apq) > 1e-17 * sqrt(fabs(app * aqq))) {
            const double tau = (aqq - app) / (2.0 * apq);
            double t;
            if (fabs(tau) > 1e150) {
              t = 0.5 / tau;
            } else {
              t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            }
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        js.pp[j] = pi;
        js.qq[j] = qi;
        js.cs[j] = c;
        js.sn[j] = s;
      }
      __syncthreads();
      // rows: C <- J^T C
      for (int e = tid; e < npairs * n; e += blockDim.x) {
        const int j = e / n, col = e - j * n;
        const double s = js.sn[j];
        if (s == 0.0) continue;
        const double c = js.cs[j];
        const int pi = js.pp[j], qi = js.qq[j];
        const double x = C[pi * ld + col], y = C[qi * ld + col];
        C[pi * ld + col] = c * x - s * y;
        C[qi * ld + col] = s * x + c * y;
      }
      __syncthreads();
      // columns: C <- C J, Q <- Q J
      for (int e = tid; e < npairs * n; e += blockDim.x) {
        const int row = e / npairs, j = e - row * npairs;
        const double s = js.sn[j];
        if (s == 0.0) continue;
        const double c = js.cs[j];
        const int pi = js.pp[j], qi = js.qq[j];
        const double x = C[row * ld + pi], y = C[row * ld + qi];
        C[row * ld + pi] = c * x - s * y;
        C[row * ld + qi] = s * x + c * y;
        const double u = Q[row * ld + pi], w = Q[row * ld + qi];
        Q[row * ld + pi] = c * u - s * w;
        Q[row * ld + qi] = s * u + c * w;
      }
      __syncthreads();
    }
  }
  return sweep;
}

// Shared tail of the polar factor: conditioning check on the Gram eigenvalues
// and M = Q diag(lambda^-1/2) Q^T written to global (ldm, zero-padded to mp).
// Returns true when lambda_min <= lambda_max / limit (or lambda_max <= 0 /
// NaN): with limit = kGramCondLimit the fit's Gram route hands the subject to
// the exact route (SRM_WARN_POLAR_CONDITION); the stateless near-orthonormal
// refinement step (k_polar_small) uses 1e24, the rank threshold of
// kernels.py:202-206 squared.
__device__ bool polar_from_eig(const double* C, const double* Q, int n, int ld, double* wsh,
                               double* M, int64_t ldm, int mp, double limit) {
  const int tid = threadIdx.x;
  __shared__ int s_bad;
  if (tid == 0) {
    double lmax = C[0], lmin = C[0];
    bool nan = false;
    for (int j = 0; j < n; ++j) {
      const double l = C[j * ld + j];
      nan |= isnan(l);
      lmax = fmax(lmax, l);
      lmin = fmin(lmin, l);
    }
    s_bad = (nan || !(lmax > 0.0) || !(lmin * limit > lmax)) ? 1 : 0;
  }
  for (int j = tid; j < n; j += blockDim.x) {
    const double l = C[j * ld + j];
    wsh[j] = l > 0.0 ? 1.0 / sqrt(l) : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < mp * mp; e += blockDim.x) {
    const int a = e / mp, b = e - a * mp;
    double m = 0.0;
    if (a < n && b < n) {
      for (int j = 0; j < n; ++j) m += (Q[a * ld + j] * Q[b * ld + j]) * wsh[j];
    }
    M[(int64_t)a * ldm + b] = m;
  }
  const bool bad = s_bad != 0;
  __syncthreads();
  return bad;
}

// init = 2: the final transform after k_ns_refine -- subjects it refined are skipped
__global__ void __launch_bounds__(kSmallThreads) k_eig_polar(DevPlan p, int init) {
  if (init == 2 && p.scal[(int64_t)(p.sub0 + blockIdx.x) * 8 + 1] != 0.0) return;
  const int iteration = init ? -1 : *p.iter;
  const int cold = (init || iteration == 0) ? 1 : 0;
  extern __shared__ __align__(16) double sm[];
  const int i = p.sub0 + blockIdx.x;
  const int n = (int)p.K;
  const int ld = n + 1;
  const int kp = (int)p.kp;
  const int np2 = (n + 1) & ~1;
  double* C = sm;
  double* Q = C + n * ld;
  double* wsh = Q + n * ld;
  double* cs = wsh + n;
  double* sn = cs + np2 / 2;
  int* pp = reinterpret_cast<int*>(sn + np2 / 2);
  int* qq = pp + np2 / 2;
  __shared__ int rot;
  const int tid = threadIdx.x;
  const double* Cg = p.bred + (int64_t)i * p.kp * p.ldo + p.ldx;
  double* Qg = p.qmat + (int64_t)i * kp * kp;
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int a = e / n, b = e - a * n;
    C[a * ld + b] = 0.5 * (Cg[(int64_t)a * p.ldo + b] + Cg[(int64_t)b * p.ldo + a]);
    Q[a * ld + b] = cold ? (a == b ? 1.0 : 0.0) : Qg[a * kp + b];
  }
  __syncthreads();
  if (!cold) {
    // rotate into the previous eigenbasis: C <- Q^T C Q (scratch in global)
    double* T1 = p.qscr + (int64_t)i * kp * kp;
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int a = e / n, b = e - a * n;
      double s = 0.0;
      for (int c = 0; c < n; ++c) s += C[a * ld + c] * Q[c * ld + b];
      T1[a * kp + b] = s;
    }
    __syncthreads();
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int a = e / n, b = e - a * n;
      double s = 0.0;
      for (int c = 0; c < n; ++c) s += Q[c * ld + a] * T1[c * kp + b];
      C[a * ld + b] = s;
    }
    __syncthreads();
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int a = e / n, b = e - a * n;
      if (a < b) {
        const double v = 0.5 * (C[a * ld + b] + C[b * ld + a]);
        C[a * ld + b] = v;
        C[b * ld + a] = v;
      }
    }
    __syncthreads();
  }
  JacobiScratch js{cs, sn, pp, qq, &rot};
  const int sweeps = jacobi_eig(C, Q, n, ld, js, 40);
  if (tid == 0) p.scal[(int64_t)i * 8 + 0] = (double)sweeps;
  const bool bad = polar_from_eig(C, Q, n, ld, wsh, p.mmat + (int64_t)i * kp * kp, kp, kp, kGramCondLimit);
  // the eigenbasis warm-starts the next iteration's sweep; the transforms of
  // init (1) and of a formed W (2) are not iterations, so they leave it alone
  // (iteration 0 starts cold anyway) and forming W mid-fit changes nothing
  if (!init)
    for (int e = tid; e < kp * kp; e += blockDim.x) {
      const int a = e / kp, b = e - a * kp;
      Qg[e] = (a < n && b < n) ? Q[a * ld + b] : 0.0;
    }
  if (bad && tid == 0) raise_warning(p.status, SRM_WARN_POLAR_CONDITION);
}

// dst[r][c] = src[r][c0 + c] (r < rows, c < cols; zero where c0 + c >= cmax),
// row pitches ldd / lds, with eight global loads in flight per thread (the
// staging of the small per-subject kernels is latency-bound otherwise)
__device__ __forceinline__ void stage_rows(double* dst, int ldd, const double* __restrict__ src, int64_t lds,
                                           int rows, int cols, int64_t c0, int64_t cmax) {
  const int total = rows * cols;
  for (int e0 = 0; e0 < total; e0 += 8 * (int)blockDim.x) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + (int)threadIdx.x + u * (int)blockDim.x;
      const int r = e / cols, c = e - r * cols;
      v[u] = (e < total && c0 + c < cmax) ? src[(int64_t)r * lds + c0 + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + (int)threadIdx.x + u * (int)blockDim.x;
      const int r = e / cols, c = e - r * cols;
      if (e < total) dst[r * ldd + c] = v[u];
    }
  }
}

// ---------------------------------------------------------------------------
// apply_m: P_i = M_i^T B_i written into the subject's term record, plus the
// per-tile cross term sum_{f,t} P[f][t] S[f][t]
// ---------------------------------------------------------------------------
// On the FP64 tensor pipe (mma.sync.m8n8k4.f64, SASS DMMA): warp w owns the
// 8-row strips f in {8 w, 8 (w + 8)}, all sixteen 8-column tiles of the
// 128-column tile; M^T (A operand) and B are staged in shared memory with row
// pitches = 4 mod 16 doubles (conflict-free fragments), the contraction over
// c < K rounded up to 4 with zero rows.

template <int NF, int COLS>
__global__ void __launch_bounds__(kSmallThreads) k_apply_m(DevPlan p, int with_cross) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double scratch[32];
  constexpr int kApplyCols = COLS;
  constexpr int kApplyLd = COLS + 4;
  constexpr int kp = 8 * NF;
  constexpr int LDM = kp + ((4 - kp) % 16 + 16) % 16;  // = 4 mod 16
  constexpr int MS = (NF + 7) / 8;                      // strips per warp
  constexpr int NT = kApplyCols / 8;
  const int tile = blockIdx.x, i = p.sub0 + blockIdx.y;
  const int K = (int)p.K;
  const int K4 = (K + 3) & ~3;
  const int64_t t0 = (int64_t)tile * kApplyCols;
  double* Ms = sm;             // [K4][LDM]: Ms[c][f] = M_i[c][f]
  double* Bs = Ms + K4 * LDM;  // [K4][kApplyLd]
  const double* Mg = p.mmat + (int64_t)i * kp * kp;
  const double* Bg = p.bred + (int64_t)i * p.kp * p.ldo;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  stage_rows(Ms, LDM, Mg, kp, K, kp, 0, K);
  stage_rows(Bs, kApplyLd, Bg, p.ldo, K, kApplyCols, t0, p.ldx);
  for (int e = tid; e < (K4 - K) * kApplyLd; e += blockDim.x) Bs[K * kApplyLd + e] = 0.0;
  for (int e = tid; e < (K4 - K) * LDM; e += blockDim.x) Ms[K * LDM + e] = 0.0;
  __syncthreads();
  double acc[MS][NT][2];
#pragma unroll
  for (int m = 0; m < MS; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  const int lr = lane >> 2, lc = lane & 3;
  for (int k0 = 0; k0 < K4; k0 += 4) {
    const double* brow = Bs + (k0 + lc) * kApplyLd + lr;
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      const int mt = w + 8 * m;
      if (mt < NF) {
        const double a = Ms[(k0 + lc) * LDM + mt * 8 + lr];  // A[f][c] = M[c][f]
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma(acc[m][n][0], acc[m][n][1], a, brow[n * 8]);
      }
    }
  }
  const int64_t* sj = p.subj + (int64_t)i * kSubjCols;
  double* P = rec_ptr(p, (int)sj[SC_SLOT]);
  double cross = 0.0;
#pragma unroll
  for (int m = 0; m < MS; ++m) {
    const int f = (w + 8 * m) * 8 + lr;
    if (w + 8 * m < NF) {
#pragma unroll
      for (int n = 0; n < NT; ++n) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t t = t0 + n * 8 + 2 * lc + h;
          if (t < p.ldx) {
            const double v = (f < K) ? acc[m][n][h] : 0.0;
            if (with_cross && f < K) cross += v * p.S[(int64_t)f * p.ldx + t];
            P[(int64_t)f * p.ldx + t] = v;
          }
        }
      }
    }
  }
  if (with_cross) {
    cross = block_sum<kSmallThreads>(cross, scratch);
    if (tid == 0) p.crossp[(int64_t)i * p.ntile_apply + tile] = cross;
  }
}

// A_i^T A_i = B_i S^T / 2 (SURVEY identity 3): CTA (chunk c, subject i) forms
// the kp x kp partial over TRs [128 c, 128 c + 128) on the FP64 tensor pipe
// (mma.sync.m8n8k4.f64: warp w owns the 8-row strips w and w + 8, all kp / 8
// column tiles), staging B and S through shared memory in two 64-TR halves
// (row pitch 68 = 4 mod 16 doubles: conflict-free fragments; 61 KB at kp = 56,
// three CTAs per SM) with eight loads in flight per thread; the last CTA of a
// subject (atomic ticket, reset after use) sums the partials in chunk order --
// deterministic -- into bred[i][a][ldx + b] (b < kp; zero for a or b >= K).
constexpr int kGfbHalf = kGfbCols / 2;
constexpr int kGfbLd = kGfbHalf + 4;

template <int KP>
__global__ void __launch_bounds__(kSmallThreads, KP <= 64 ? 3 : 1) k_gram_from_b(DevPlan p) {
  extern __shared__ __align__(16) double sm[];
  constexpr int NT = KP / 8;
  constexpr int MS = (NT + 7) / 8;
  const int c = blockIdx.x, i = p.sub0 + blockIdx.y;
  const int K = (int)p.K;
  double* Bs = sm;              // [KP][kGfbLd], rows >= K zero
  double* Ss = sm + KP * kGfbLd;
  const double* Bg = p.bred + (int64_t)i * p.kp * p.ldo;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  for (int e = tid; e < (KP - K) * kGfbLd; e += blockDim.x) {
    Bs[K * kGfbLd + e] = 0.0;
    Ss[K * kGfbLd + e] = 0.0;
  }
  double acc[MS][NT][2];
#pragma unroll
  for (int m = 0; m < MS; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
  for (int h = 0; h < 2; ++h) {
    const int64_t t0 = (int64_t)c * kGfbCols + h * kGfbHalf;
    if (h) __syncthreads();  // the first half's reads are done
    stage_rows(Bs, kGfbLd, Bg, p.ldo, K, kGfbHalf, t0, p.ldx);
    stage_rows(Ss, kGfbLd, p.S, p.ldx, K, kGfbHalf, t0, p.ldx);
    __syncthreads();
#pragma unroll 2
    for (int k0 = 0; k0 < kGfbHalf; k0 += 4) {
#pragma unroll
      for (int m = 0; m < MS; ++m) {
        const int mt = w + 8 * m;
        if (mt < NT) {
          const double a = Bs[(mt * 8 + lr) * kGfbLd + k0 + lc];  // A[a][t] = B[a][t]
#pragma unroll
          for (int n = 0; n < NT; ++n)                            // B[t][b] = S[b][t]
            dmma(acc[m][n][0], acc[m][n][1], a, Ss[(n * 8 + lr) * kGfbLd + k0 + lc]);
        }
      }
    }
  }
  constexpr int kp = KP;
  double* part = p.gfb_part + ((int64_t)i * p.gfb_chunks + c) * kp * kp;
#pragma unroll
  for (int m = 0; m < MS; ++m) {
    const int mt = w + 8 * m;
    if (mt < NT) {
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        double* d = part + (mt * 8 + lr) * kp + n * 8 + 2 * lc;
        d[0] = acc[m][n][0];
        d[1] = acc[m][n][1];
      }
    }
  }
  // last CTA of subject i reduces
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(p.gfb_count + i, 1) == p.gfb_chunks - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // 16 elements per thread per batch: each chunk step issues 16 independent
  // L2 loads (summation order over chunks unchanged); ld_cg, not __ldcg,
  // whose strong loads the compiler keeps in order, a few in flight
  const double* all = p.gfb_part + (int64_t)i * p.gfb_chunks * kp * kp;
  double* out = p.bred + (int64_t)i * p.kp * p.ldo + p.ldx;
  const int n = kp * kp;
  for (int e0 = 0; e0 < n; e0 += 16 * (int)blockDim.x) {
    double s[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) s[u] = 0.0;
    for (int q = 0; q < p.gfb_chunks; ++q) {
      const double* src = all + (int64_t)q * n;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = e0 + tid + u * (int)blockDim.x;
        if (e < n) s[u] += ld_cg(src + e);
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = e0 + tid + u * (int)blockDim.x;
      if (e < n) out[(int64_t)(e / kp) * p.ldo + e % kp] = 0.5 * s[u];
    }
  }
  if (tid == 0) p.gfb_count[i] = 0;
}

// ---------------------------------------------------------------------------
// SRM_FLAG_COLBLOCK: the ordered accumulation of srm.py:193-213 by TR column
// blocks.  pack: local record j's columns [q xw, (q + 1) xw) (and its scalars)
// -> xsend[q][j]; after the all-to-all, xrecv[r][j] holds rank r's subject j
// for this rank's block.  reduce: the same left fold as k_reduce_terms over
// (r, j) = ascending global subject order (ranks own contiguous shards,
// cli.py:82-85), so the block equals one rank's sum bit for bit.  unpack: the
// all-gathered blocks -> red.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads) k_xchg_pack(DevPlan p) {
  const int j = blockIdx.y, q = blockIdx.z;
  const int64_t e = (int64_t)blockIdx.x * kSmallThreads + threadIdx.x;
  if (e >= p.xrec) return;
  const int64_t* sj = p.subj + (int64_t)j * kSubjCols;
  const double* rec = rec_ptr(p, (int)sj[SC_SLOT]);
  const int64_t kx = p.kp * p.xw;
  double v;
  if (e < kx) {
    const int64_t f = e / p.xw, col = (int64_t)q * p.xw + (e - f * p.xw);
    v = col < p.ldx ? rec[f * p.ldx + col] : 0.0;
  } else {
    v = rec[p.kp * p.ldx + (e - kx)];
  }
  p.xsend[((int64_t)q * p.max_local + j) * p.xrec + e] = v;
}

__global__ void __launch_bounds__(kSmallThreads) k_xchg_reduce(DevPlan p) {
  const int64_t kx = p.kp * p.xw;
  const int64_t e = (int64_t)blockIdx.x * kSmallThreads + threadIdx.x;
  double* out = p.xredbuf + (int64_t)p.rank * p.xred;
  if (e < kx) {
    double acc = 0.0;
    bool first = true;
    for (int r = 0; r < p.world; ++r) {
      const double* base = p.xrecv + (int64_t)r * p.max_local * p.xrec;
      const int cnt = p.xcounts[r];
      int j = 0;
      for (; j + 8 <= cnt; j += 8) {  // eight loads in flight, summed in order
        double x[8], rr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          x[u] = base[(int64_t)(j + u) * p.xrec + e];
          rr[u] = base[(int64_t)(j + u) * p.xrec + kx + RC_RHO2];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc = first ? x[u] / rr[u] : acc + x[u] / rr[u];
          first = false;
        }
      }
      for (; j < cnt; ++j) {
        const double v = base[(int64_t)j * p.xrec + e] / base[(int64_t)j * p.xrec + kx + RC_RHO2];
        acc = first ? v : acc + v;
        first = false;
      }
    }
    out[e] = acc;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // the scalar sums of k_reduce_terms, same order
    double rho0 = 0.0, vlog = 0.0, sq = 0.0, vsum = 0.0;
    bool first = true;
    for (int r = 0; r < p.world; ++r) {
      const double* base = p.xrecv + (int64_t)r * p.max_local * p.xrec + kx;
      for (int j = 0; j < p.xcounts[r]; ++j) {
        const double* sc = base + (int64_t)j * p.xrec;
        const double rr = sc[RC_RHO2];
        rho0 = first ? 1.0 / rr : rho0 + 1.0 / rr;
        first = false;
        vlog += sc[RC_V] * log(rr);
        sq += sc[RC_SQNORM] / rr;
        vsum += sc[RC_V];
      }
    }
    out[kx + RD_RHO0] = rho0;
    out[kx + RD_VLOGRHO] = vlog;
    out[kx + RD_SQRHO] = sq;
    out[kx + RD_VSUM] = vsum;
  }
}

__global__ void __launch_bounds__(kSmallThreads) k_xchg_unpack(DevPlan p) {
  const int q = blockIdx.y;
  const int64_t kx = p.kp * p.xw;
  const int64_t e = (int64_t)blockIdx.x * kSmallThreads + threadIdx.x;
  const double* src = p.xredbuf + (int64_t)q * p.xred;
  if (e < kx) {
    const int64_t f = e / p.xw, col = (int64_t)q * p.xw + (e - f * p.xw);
    if (col < p.ldx) p.red[f * p.ldx + col] = src[e];
  } else if (q == p.rank && e < kx + kRedScalars) {
    p.red[p.kp * p.ldx + (e - kx)] = src[e];
  }
}

__device__ __forceinline__ int64_t hist_row(const DevPlan& p, int it) { return (int64_t)(it % p.n_hist) * p.hist_stride; }

__global__ void k_set_iteration(DevPlan p, int iteration, int advance) {
  if (advance) *p.iter += 1;
  else *p.iter = iteration;
}

// advance (single-block launches): thread 0 then moves the device iteration
// counter on, after every thread has read it
__global__ void k_finalize_rho(DevPlan p, int init, int advance) {
  const int iteration = init ? -1 : *p.iter;
  if (advance) {
    __syncthreads();
    if (threadIdx.x == 0) *p.iter = iteration + 1;
  }
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= p.nsub) return;
  const int i = p.sub0 + w;
  const int64_t* sj = p.subj + (int64_t)i * kSubjCols;
  double* rec = rec_ptr(p, (int)sj[SC_SLOT]) + p.kp * p.ldx;
  double rho2 = 1.0;
  if (!init) {
    double cross = 0.0;
    for (int t = 0; t < p.ntile_apply; ++t) cross += p.crossp[(int64_t)i * p.ntile_apply + t];
    const double T = (double)p.T;
    const double trace = p.tailscr[TS_TRACE];
    rho2 = (rec[RC_SQNORM] + T * trace - 2.0 * cross) / (T * rec[RC_V]);
    rho2 = fmax(rho2, 1e-12);
    if (iteration >= 0) p.hist[hist_row(p, iteration) + SRM_H_RHO2 + i] = rho2;
  }
  rec[RC_RHO2] = rho2;
}

// ---------------------------------------------------------------------------
// reduce_terms: dst = sum_j rec[order[j]] / rho2_j, ascending order
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads) k_reduce_terms(DevPlan p, double* dst,
                                                                const int32_t* __restrict__ order,
                                                                int count, int ident) {
  const int64_t n = p.kp * p.ldx;
  const int64_t e = (int64_t)blockIdx.x * kSmallThreads + threadIdx.x;
  if (e < n) {
    // subjects in `order`, summed sequentially; loads batched 16 deep (the
    // per-subject rho^2 are the same for every element: L1 broadcasts)
    double acc = 0.0;
    int j = 0;
    for (; j + 16 <= count; j += 16) {
      double x[16], r[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const double* rec = rec_ptr(p, ident ? j + u : order[j + u]);
        x[u] = rec[e];
        r[u] = rec[n + RC_RHO2];
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = (j + u == 0) ? x[u] / r[u] : acc + x[u] / r[u];
    }
    for (; j + 4 <= count; j += 4) {
      double x[4], r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* rec = rec_ptr(p, ident ? j + u : order[j + u]);
        x[u] = rec[e];
        r[u] = rec[n + RC_RHO2];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = (j + u == 0) ? x[u] / r[u] : acc + x[u] / r[u];
    }
    for (; j < count; ++j) {
      const double* rec = rec_ptr(p, ident ? j : order[j]);
      const double v = rec[e] / rec[n + RC_RHO2];
      acc = (j == 0) ? v : acc + v;
    }
    dst[e] = acc;
  }
  if (blockIdx.x == 0) {
    // per-subject scalar terms in parallel, then one thread sums them in order
    __shared__ double terms[4][kSmallThreads];
    double rho0 = 0.0, vlog = 0.0, sq = 0.0, vsum = 0.0;
    for (int j0 = 0; j0 < count; j0 += kSmallThreads) {
      const int j = j0 + (int)threadIdx.x;
      if (j < count) {
        const double* rec = rec_ptr(p, order[j]) + n;
        const double r = rec[RC_RHO2];
        terms[0][threadIdx.x] = 1.0 / r;
        terms[1][threadIdx.x] = rec[RC_V] * log(r);
        terms[2][threadIdx.x] = rec[RC_SQNORM] / r;
        terms[3][threadIdx.x] = rec[RC_V];
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const int m = min(kSmallThreads, count - j0);
        for (int u = 0; u < m; ++u) {
          rho0 = (j0 + u == 0) ? terms[0][u] : rho0 + terms[0][u];
          vlog += terms[1][u];
          sq += terms[2][u];
          vsum += terms[3][u];
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      dst[n + RD_RHO0] = rho0;
      dst[n + RD_VLOGRHO] = vlog;
      dst[n + RD_SQRHO] = sq;
      dst[n + RD_VSUM] = vsum;
    }
  }
}
// In-place inverse of an SPD n x n matrix (n <= 128) by the symmetric sweep
// (Gauss-Jordan without pivoting), register-resident: a 16 x 16 thread grid
// owns the cyclic R x R blocks a[i][k] = A[ty + 16 i][tx + 16 k]
// (R = ceil(n / 16)), and each pivot step broadcasts only the pivot row
// through a double-buffered shared vector (one barrier per step).  The pivot
// at step j is the LDL^T pivot d_j (the square of Cholesky's L_jj), so
// logdet = sum log d_j and the first non-positive pivot is the index scipy's
// cho_factor reports (kernels.py:168-187).  Sweeping every pivot leaves
// -A^{-1} in a.  Returns the failed pivot or -1; d_j lands in dbuf[j].
constexpr int kSweepLd = 128;

struct SweepShared {
  double pbuf[2 * kSweepLd];  // double-buffered pivot row
  double dbuf[kSweepLd];      // pivots
  double scratch[32];
};

template <int R>
__device__ __forceinline__ void reg_load(double (&a)[R][R], const double* src, int64_t lds, int n) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int r = ty + 16 * i, c = tx + 16 * k;
      a[i][k] = (r < n && c < n) ? src[r * lds + c] : 0.0;
    }
}

// Row / column s = j / 16 of the thread's register block by a compile-time
// index (a runtime index would put a[][] in local memory): the switch on s is
// warp-uniform, and inside it the owners of row j / column j / the pivot take
// their new values by selects -- 3R selects per thread and pivot where a
// select per element cost R^2, and no divergent branch.
template <int R, int S>
__device__ __forceinline__ void sweep_fix(double (&a)[R][R], const double* pr, const double* pc, double inv,
                                          bool row_owner, bool col_owner) {
  if constexpr (S < R) {
#pragma unroll
    for (int k = 0; k < R; ++k) a[S][k] = row_owner ? pc[k] * inv : a[S][k];
#pragma unroll
    for (int i = 0; i < R; ++i) a[i][S] = col_owner ? pr[i] : a[i][S];
    a[S][S] = (row_owner && col_owner) ? -inv : a[S][S];
  }
}
template <int R, int S>
__device__ __forceinline__ void sweep_put_row(const double (&a)[R][R], double* nx, int tx, int n) {
  if constexpr (S < R) {
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (tx + 16 * k < n) nx[tx + 16 * k] = a[S][k];
  }
}

template <int R>
__device__ __forceinline__ int reg_sweep(double (&a)[R][R], int n, double* pbuf, double* dbuf) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  if (ty == 0) {
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (tx + 16 * k < n) pbuf[tx + 16 * k] = a[0][k];
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double* pv = pbuf + (j & 1) * kSweepLd;
    const double d = pv[j];
    if (!(d > 0.0)) return j;  // uniform: every thread reads the same pivot
    const double inv = 1.0 / d;
    double pr[R], pc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = ty + 16 * i;
      pr[i] = (r < n) ? pv[r] * inv : 0.0;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int c = tx + 16 * k;
      pc[k] = (c < n) ? pv[c] : 0.0;
    }
    // every element as if off the pivot row and column (one FMA each), then
    // row j (pv[c] / d), column j (pv[r] / d) and the pivot (-1 / d) written
    // over it by their owners -- the values of the per-element select form
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int k = 0; k < R; ++k) a[i][k] = fma(-pr[i], pc[k], a[i][k]);
    const int jr = j & 15;
    const bool row_owner = ty == jr, col_owner = tx == jr;
    switch (j >> 4) {
      case 0: sweep_fix<R, 0>(a, pr, pc, inv, row_owner, col_owner); break;
      case 1: sweep_fix<R, 1>(a, pr, pc, inv, row_owner, col_owner); break;
      case 2: sweep_fix<R, 2>(a, pr, pc, inv, row_owner, col_owner); break;
      case 3: sweep_fix<R, 3>(a, pr, pc, inv, row_owner, col_owner); break;
      case 4: sweep_fix<R, 4>(a, pr, pc, inv, row_owner, col_owner); break;
      case 5: sweep_fix<R, 5>(a, pr, pc, inv, row_owner, col_owner); break;
      case 6: sweep_fix<R, 6>(a, pr, pc, inv, row_owner, col_owner); break;
      default: sweep_fix<R, 7>(a, pr, pc, inv, row_owner, col_owner); break;
    }
    if (threadIdx.x == 0) dbuf[j] = d;
    const int jn = j + 1;
    if (jn < n && ty == (jn & 15)) {
      double* nx = pbuf + (jn & 1) * kSweepLd;
      switch (jn >> 4) {
        case 0: sweep_put_row<R, 0>(a, nx, tx, n); break;
        case 1: sweep_put_row<R, 1>(a, nx, tx, n); break;
        case 2: sweep_put_row<R, 2>(a, nx, tx, n); break;
        case 3: sweep_put_row<R, 3>(a, nx, tx, n); break;
        case 4: sweep_put_row<R, 4>(a, nx, tx, n); break;
        case 5: sweep_put_row<R, 5>(a, nx, tx, n); break;
        case 6: sweep_put_row<R, 6>(a, nx, tx, n); break;
        default: sweep_put_row<R, 7>(a, nx, tx, n); break;
      }
    }
    __syncthreads();
  }
  return -1;
}

// sum_j log d_j in a fixed tree order (all threads get it)
__device__ double sum_log(const double* dbuf, int n, double* scratch) {
  const double v = ((int)threadIdx.x < n) ? log(dbuf[threadIdx.x]) : 0.0;
  return block_sum<kSmallThreads>(v, scratch);
}

// ---------------------------------------------------------------------------
// tail, stage 0 (one CTA): -Sigma_s^{-1} and log det Sigma_s (srm.py:127 inner
// spd_inverse).  Sigma_s is final after k_tail_sigma, so the next E-step's
// inverse runs on a side stream while the M-step of this iteration does.
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void tail_inv_body(const DevPlan& p, SweepShared& sh) {
  const int n = (int)p.K, kp = (int)p.kp;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double a[R][R];
  reg_load<R>(a, p.sigma, kp, n);
  const int piv = reg_sweep<R>(a, n, sh.pbuf, sh.dbuf);  // a = -Sigma_s^{-1}
  if (piv >= 0) {
    if (tid == 0) raise_status(p.status, SRM_ERR_DEFINITENESS, piv, -1);
    return;
  }
  const double logdet_sigma = sum_log(sh.dbuf, n, sh.scratch);
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int r = ty + 16 * i, c = tx + 16 * k;
      if (r < n && c < n) p.sinv[r * kp + c] = a[i][k];
    }
  if (tid == 0) p.tailscr[TS_LOGDET_SIGMA] = logdet_sigma;
}

template <int R>
__global__ void __launch_bounds__(kSmallThreads) k_tail_inv(DevPlan p) {
  __shared__ SweepShared sh;
  if (failed(p)) return;
  tail_inv_body<R>(p, sh);
}

// ---------------------------------------------------------------------------
// tail, stage 1 (one CTA): var_s = (rho0 I + Sigma_s^{-1})^{-1} and
// C = Sigma_s^T (I - rho0 var_s) = var_s (srm.py:127-128).  rho0 = sum 1 / rho_j^2 in
// ascending order straight from the term table (ordered plans: the same sum
// k_reduce_terms forms, so this stage runs beside it), else from `red`.
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void tail_kk_body(const DevPlan& p, int iteration, SweepShared& sh) {
  double* pbuf = sh.pbuf;
  double* dbuf = sh.dbuf;
  const int n = (int)p.K, kp = (int)p.kp;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  __shared__ double s_rho0;
  double a[R][R];
  reg_load<R>(a, p.sinv, kp, n);  // -Sigma_s^{-1} (k_tail_inv)
  if (p.flags & SRM_FLAG_ORDERED) {
    // 1 / rho_j^2 loaded in parallel, summed by one thread in ascending order
    double* rinv = sh.pbuf;
    const int64_t nrec = p.kp * p.ldx;
    double rho0 = 0.0;
    for (int j0 = 0; j0 < p.n_order; j0 += 2 * kSweepLd) {
      const int m = min(2 * kSweepLd, p.n_order - j0);
      for (int u = tid; u < m; u += blockDim.x) rinv[u] = 1.0 / rec_ptr(p, p.order[j0 + u])[nrec + RC_RHO2];
      __syncthreads();
      if (tid == 0)
        for (int u = 0; u < m; ++u) rho0 = (j0 + u == 0) ? rinv[u] : rho0 + rinv[u];
      __syncthreads();
    }
    if (tid == 0) s_rho0 = rho0;
  } else if (tid == 0) {
    s_rho0 = p.red[p.kp * p.ldx + RD_RHO0];
  }
  __syncthreads();
  const double rho0 = s_rho0;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int r = ty + 16 * i, c = tx + 16 * k;
      a[i][k] = (r < n && c < n) ? (r == c ? rho0 : 0.0) - a[i][k] : 0.0;
    }
  const int piv = reg_sweep<R>(a, n, pbuf, dbuf);  // a = -var_s
  if (piv >= 0) {
    if (tid == 0) raise_status(p.status, SRM_ERR_DEFINITENESS, piv, iteration);
    return;
  }
  const double logdet_prec = sum_log(dbuf, n, sh.scratch);
  // C = Sigma_s^T (I - rho0 var_s) (srm.py:128) is var_s itself: Sigma_s and
  // var_s = (Sigma_s^{-1} + rho0 I)^{-1} = Sigma_s (I + rho0 Sigma_s)^{-1}
  // commute, and var_s (Sigma_s^{-1} + rho0 I) = I gives var_s = Sigma_s -
  // rho0 Sigma_s var_s = Sigma_s (I - rho0 var_s).  Taking var_s also skips
  // the cancellation in I - rho0 var_s (~1 / (1 + rho0 lambda)) and the K^3
  // product on the critical path; the two differ by rounding only (~eps
  // cond(Sigma_s^{-1} + rho0 I)).
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int r = ty + 16 * i, c = tx + 16 * k;
      if (r < kp && c < kp) {
        const double v = (r < n && c < n) ? -a[i][k] : 0.0;
        p.var[r * kp + c] = v;
        p.cmat[r * kp + c] = v;
      }
    }
  if (tid == 0) p.tailscr[TS_LOGDET_PREC] = logdet_prec;
}

template <int R>
__global__ void __launch_bounds__(kSmallThreads) k_tail_kk(DevPlan p) {
  __shared__ SweepShared sh;
  const int iteration = *p.iter;
  if (failed(p)) return;
  tail_kk_body<R>(p, iteration, sh);
}

// tail, stage 2 (32-column tiles): S = C red, quad = <red, var red>, S S^T
// partials and the tolerance statistics.
// sixteen warps: each row chain (a K-long dependent FMA sequence per
// accumulator) is short of issue slots at two warps per scheduler
constexpr int kTailSThreads = 512;
__global__ void __launch_bounds__(kTailSThreads) k_tail_s(DevPlan p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double scratch[32];
  if (failed(p)) return;
  const int K = (int)p.K, kp = (int)p.kp;
  const int tile = blockIdx.x;
  const int64_t t0 = (int64_t)tile * 32;
  constexpr int LD = 33;  // padded rows: conflict-free S S^T reads
  double* Rt = sm;           // [K][33]
  double* St = sm + K * LD;  // [K][33]
  double* So = St + K * LD;  // [K][33] S before this E-step (tolerance statistic)
  const int tid = threadIdx.x, col = tid & 31, rg = tid >> 5;
  const int64_t t = t0 + col;
  const bool tin = t < p.ldx;
  stage_rows(Rt, LD, p.red, p.ldx, K, 32, t0, p.ldx);
  stage_rows(So, LD, p.S, p.ldx, K, 32, t0, p.ldx);
  __syncthreads();
  double quad = 0.0, dsq = 0.0, osq = 0.0;
  // rows f of C and var_s, one coalesced load per warp, broadcast by shuffles;
  // the next row's loads are issued before this row's products
  double cm[4], vr[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = q * 32 + col;
    cm[q] = (c < K && rg < K) ? p.cmat[rg * kp + c] : 0.0;
    vr[q] = (c < K && rg < K) ? p.var[rg * kp + c] : 0.0;
  }
  for (int f = rg; f < K; f += kTailSThreads / 32) {
    double cmn[4], vrn[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = q * 32 + col;
      cmn[q] = (c < K && f + kTailSThreads / 32 < K) ? p.cmat[(f + kTailSThreads / 32) * kp + c] : 0.0;
      vrn[q] = (c < K && f + kTailSThreads / 32 < K) ? p.var[(f + kTailSThreads / 32) * kp + c] : 0.0;
    }
    double s = 0.0, y = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int lmax = min(32, K - q * 32);
      if (lmax <= 0) break;
#pragma unroll 8
      for (int l = 0; l < lmax; ++l) {
        const double r = Rt[(q * 32 + l) * LD + col];
        s += __shfl_sync(0xffffffffu, cm[q], l) * r;
        y += __shfl_sync(0xffffffffu, vr[q], l) * r;
      }
    }
    quad += Rt[f * LD + col] * y;
    St[f * LD + col] = s;
    if (tin && p.st) p.st[t * kp + f] = s;
    if (tin && p.sf) {
      const float sfv = (float)s;
      const float hi = __uint_as_float(__float_as_uint(sfv) & 0xFFFFE000u);
      p.sf[(int64_t)f * p.ldx + t] = hi;
      p.sf[(int64_t)(p.np + f) * p.ldx + t] = sfv - hi;
    }
    if (tin) {
      const double old = So[f * LD + col];
      dsq += (s - old) * (s - old);
      osq += old * old;
      p.S[(int64_t)f * p.ldx + t] = s;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cm[q] = cmn[q];
      vr[q] = vrn[q];
    }
  }
  __syncthreads();
  double* ssp = p.sspart + (int64_t)tile * kp * kp;
  for (int e = tid; e < K * K; e += blockDim.x) {
    const int a = e / K, b = e - a * K;
    if (a > b) continue;  // symmetric: the product commutes exactly
    double v = 0.0;
#pragma unroll 8
    for (int c = 0; c < 32; ++c) v += St[a * LD + c] * St[b * LD + c];
    ssp[a * kp + b] = v;
    ssp[b * kp + a] = v;
  }
  quad = block_sum<kTailSThreads>(quad, scratch);
  dsq = block_sum<kTailSThreads>(dsq, scratch);
  osq = block_sum<kTailSThreads>(osq, scratch);
  if (tid == 0) {
    p.tailpart[tile * 4 + 0] = quad;
    p.tailpart[tile * 4 + 1] = dsq;
    p.tailpart[tile * 4 + 2] = osq;
  }
}

// tail, stage 3 (one CTA): Sigma_s <- sym(var_s + S S^T / T), trace, LL
constexpr int kSigmaThreads = 1024;
__global__ void __launch_bounds__(kSigmaThreads) k_tail_sigma(DevPlan p) {
  const int iteration = *p.iter;
  extern __shared__ __align__(16) double sm[];
  if (failed(p)) return;
  const int K = (int)p.K, kp = (int)p.kp, nt = p.ntile_tail;
  const int tid = threadIdx.x;
  const double T = (double)p.T;
  double* Sn = sm;           // [K][K]
  double* tp = sm + K * K;   // [nt][4] tile statistics
  for (int e = tid; e < nt * 4; e += blockDim.x) tp[e] = p.tailpart[e];
  const int64_t tstride = (int64_t)kp * kp;
  for (int e = tid; e < K * K; e += blockDim.x) {
    const int a = e / K, b = e - a * K;
    const double* src = p.sspart + a * kp + b;
    double ss = 0.0;
    int tile = 0;
    for (; tile + 8 <= nt; tile += 8) {  // 8 loads in flight, summed in tile order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = src[(tile + u) * tstride];
#pragma unroll
      for (int u = 0; u < 8; ++u) ss += v[u];
    }
    for (; tile < nt; ++tile) ss += src[tile * tstride];
    Sn[e] = p.var[a * kp + b] + ss / T;
  }
  __syncthreads();
  for (int e = tid; e < K * K; e += blockDim.x) {
    const int a = e / K, b = e - a * K;
    p.sigma[a * kp + b] = 0.5 * (Sn[a * K + b] + Sn[b * K + a]);
  }
  if (tid == 0) {
    double trace = 0.0;
    for (int a = 0; a < K; ++a) trace += 0.5 * (Sn[a * K + a] + Sn[a * K + a]);
    double quad = 0.0, dsq = 0.0, osq = 0.0;
    for (int tile = 0; tile < nt; ++tile) {
      quad += tp[tile * 4 + 0];
      dsq += tp[tile * 4 + 1];
      osq += tp[tile * 4 + 2];
    }
    const double* rs = p.red + p.kp * p.ldx;
    const double two_pi = 6.283185307179586476925286766559;
    const double ll = -0.5 * (T * (rs[RD_VSUM] * log(two_pi) + rs[RD_VLOGRHO] +
                                   p.tailscr[TS_LOGDET_SIGMA] + p.tailscr[TS_LOGDET_PREC]) +
                              (rs[RD_SQRHO] - quad));
    double* h = p.hist + hist_row(p, iteration);
    h[SRM_H_LL] = ll;
    h[SRM_H_TRACE] = trace;
    h[SRM_H_RHO0] = rs[RD_RHO0];
    h[SRM_H_SDIFF] = sqrt(dsq);
    h[SRM_H_SPREV] = sqrt(osq);
    p.tailscr[TS_TRACE] = trace;
  }
}

// mirror the computed upper triangle of every X_i^T X_i into the lower one
__global__ void k_mirror_gram(DevPlan p, int first) {
  const int64_t n = p.ldx * p.ldx;
  double* g = p.gram + (int64_t)(first + blockIdx.y) * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e / p.ldx, b = e - a * p.ldx;
    if (a > b) g[e] = g[b * p.ldx + a];
  }
}

// restart the EM state: Sigma_s = I (srm.py:248), clear the status word and
// the iteration counter
__global__ void k_reset(DevPlan p) {
  const int kp = (int)p.kp;
  for (int e = threadIdx.x; e < kp * kp; e += blockDim.x) {
    const int a = e / kp, b = e - a * kp;
    p.sigma[e] = (a == b && a < p.K) ? 1.0 : 0.0;
    p.sinv[e] = (a == b && a < p.K) ? -1.0 : 0.0;  // the sweep of I
  }
  if (threadIdx.x == 0) {
    p.status[0] = p.status[1] = p.status[2] = p.status[3] = 0;
    *p.iter = 0;
    p.tailscr[TS_LOGDET_SIGMA] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// apply_w: W_i[r][f] = sum_c A_i[r][c] M_i[c][f]  (row tiles of 128)
// ---------------------------------------------------------------------------
// fp32 A (tensor-core path): item o_off indexes the [rows][np] fp32 A region
__global__ void __launch_bounds__(kSmallThreads) k_apply_w_f32(DevPlan p, const ItemA* __restrict__ items) {
  extern __shared__ __align__(16) double sm[];
  const ItemA it = items[blockIdx.x];
  const int i = it.pad;
  const int K = (int)p.K, kp = (int)p.kp;
  const double* Mg = p.mmat + (int64_t)i * kp * kp;
  double* Ms = sm;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) Ms[e] = Mg[(e / K) * kp + e % K];
  __syncthreads();
  const int64_t row0 = it.x_off / p.ldx;
  for (int e = threadIdx.x; e < it.rows * K; e += blockDim.x) {
    const int r = e / K, f = e - r * K;
    const float* a = p.af + (row0 + r) * p.np;
    double s = 0.0;
    for (int c = 0; c < K; ++c) s += (double)a[c] * Ms[c * K + f];
    p.wout[(row0 + r) * K + f] = s;
  }
}

__global__ void __launch_bounds__(kSmallThreads) k_apply_w(DevPlan p, const ItemA* __restrict__ items) {
  extern __shared__ __align__(16) double sm[];
  const ItemA it = items[blockIdx.x];
  const int i = it.pad;
  const int K = (int)p.K, kp = (int)p.kp;
  const double* Mg = p.mmat + (int64_t)i * kp * kp;
  double* Ms = sm;  // [K][K]
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) Ms[e] = Mg[(e / K) * kp + e % K];
  __syncthreads();
  const int64_t row0 = it.o_off / kp;  // A row index of the tile start
  for (int e = threadIdx.x; e < it.rows * K; e += blockDim.x) {
    const int r = e / K, f = e - r * K;
    const double* a = p.amat + (row0 + r) * kp;
    double s = 0.0;
    for (int c = 0; c < K; ++c) s += a[c] * Ms[c * K + f];
    p.wout[(row0 + r) * K + f] = s;
  }
}

// ---------------------------------------------------------------------------
// stateless: in-place SPD inverse (kernels.py:168-187)
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void spd_inverse_body(double* g, int n, int32_t* status, SweepShared& sh) {
  double* pbuf = sh.pbuf;
  double* dbuf = sh.dbuf;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double a[R][R];
  reg_load<R>(a, g, n, n);
  const int piv = reg_sweep<R>(a, n, pbuf, dbuf);
  if (piv >= 0) {
    if (threadIdx.x == 0) raise_status(status, SRM_ERR_DEFINITENESS, piv, -1);
    return;
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int r = ty + 16 * i, c = tx + 16 * k;
      // the lower triangle, mirrored: kernels.py:185-187 symmetrizes dpotri's
      // lower factor exactly (tril + tril(-1)^T), so the result equals its transpose
      if (r < n && c < n && r >= c) {
        g[r * n + c] = -a[i][k];
        g[c * n + r] = -a[i][k];
      }
    }
}

template <int R>
__global__ void __launch_bounds__(kSmallThreads) k_spd_inverse(double* a, int n, int32_t* status) {
  __shared__ SweepShared sh;
  spd_inverse_body<R>(a, n, status, sh);
}

// stateless polar transform from a Gram matrix: M = G^{-1/2}
__global__ void __launch_bounds__(kSmallThreads) k_polar_small(const double* g, int64_t ldg, int n,
                                                               double* m, int64_t ldm, int32_t* status) {
  extern __shared__ __align__(16) double sm[];
  const int ld = n + 1;
  const int np2 = (n + 1) & ~1;
  double* C = sm;
  double* Q = C + n * ld;
  double* wsh = Q + n * ld;
  double* cs = wsh + n;
  double* sn = cs + np2 / 2;
  int* pp = reinterpret_cast<int*>(sn + np2 / 2);
  int* qq = pp + np2 / 2;
  __shared__ int rot;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int a = e / n, b = e - a * n;
    C[a * ld + b] = 0.5 * (g[a * ldg + b] + g[b * ldg + a]);
    Q[a * ld + b] = a == b ? 1.0 : 0.0;
  }
  __syncthreads();
  JacobiScratch js{cs, sn, pp, qq, &rot};
  jacobi_eig(C, Q, n, ld, js, 40);
  const bool bad = polar_from_eig(C, Q, n, ld, wsh, m, ldm, n, 1e24);
  if (bad && threadIdx.x == 0) raise_status(status, SRM_ERR_RANK, 0, -1);
}

__global__ void __launch_bounds__(kSmallThreads) k_apply_right(const double* a, int64_t lda, int64_t v, int k,
                                                               const double* m, int64_t ldm, double* w,
                                                               int64_t ldw) {
  extern __shared__ __align__(16) double sm[];
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) sm[e] = m[(e / k) * ldm + e % k];
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  for (int e = threadIdx.x; e < 64 * k; e += blockDim.x) {
    const int64_t r = r0 + e / k;
    const int f = e % k;
    if (r >= v) continue;
    double s = 0.0;
    for (int c = 0; c < k; ++c) s += a[r * lda + c] * sm[c * k + f];
    w[r * ldw + f] = s;
  }
}

size_t eig_smem_bytes(int n) {
  const int np2 = (n + 1) & ~1;
  return (size_t)(2 * n * (n + 1) + n + np2) * sizeof(double) + (size_t)np2 * sizeof(int);
}

// Raise a kernel's dynamic smem limit once (never inside a graph capture after
// the first eager launch of the same shape).
// Raise a kernel's dynamic shared-memory limit once (static + dynamic may not
// exceed 48 KB without it); cached per function.
cudaError_t set_smem(const void* f, size_t bytes) {
  if (bytes <= 16 * 1024) return cudaSuccess;
  static const void* funcs[64];
  static size_t limits[64];
  static int n = 0;
  for (int i = 0; i < n; ++i) {
    if (funcs[i] == f) {
      if (bytes <= limits[i]) return cudaSuccess;
      cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
      if (e == cudaSuccess) limits[i] = bytes;
      return e;
    }
  }
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && n < 64) {
    funcs[n] = f;
    limits[n] = bytes;
    ++n;
  }
  return e;
}

}  // namespace

int max_supported_k() { return kMaxK; }

cudaError_t launch_prep(const DevPlan& p, int local, int64_t V, const void* x, int x_dtype,
                        int64_t ld, int xhat_dtype, cudaStream_t s) {
  const dim3 grid((unsigned)((V + kPrepRows - 1) / kPrepRows));
  if (V == 0) return cudaSuccess;
  size_t smem = 0;
  if (p.cmax) {  // fresh column maxima for this subject
    cudaError_t e = cudaMemsetAsync(p.cmax + (int64_t)local * p.ldx, 0, (size_t)p.ldx * 8, s);
    if (e != cudaSuccess) return e;
    smem = (size_t)p.ldx * 8;
  }
  const void* fn = nullptr;
  if (x_dtype == SRM_F64 && xhat_dtype == SRM_F64) fn = (const void*)k_prep<double, double>;
  else if (x_dtype == SRM_F64 && xhat_dtype == SRM_F32) fn = (const void*)k_prep<double, float>;
  else if (x_dtype == SRM_F32 && xhat_dtype == SRM_F32) fn = (const void*)k_prep<float, float>;
  else fn = (const void*)k_prep<float, double>;
  cudaError_t e = set_smem(fn, smem);
  if (e != cudaSuccess) return e;
  DevPlan arg = p;
  void* args[] = {&arg, &local, &x, &ld};
  e = cudaLaunchKernel(fn, grid, dim3(kSmallThreads), args, smem, s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_subject_sqnorm(const DevPlan& p, cudaStream_t s) {
  k_subject_sqnorm<<<p.n_local, kSmallThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_reduce_chunks(const DevPlan& p, cudaStream_t s) {
  const int64_t n2 = p.kp * p.ldo / 2;
  const dim3 grid((unsigned)((n2 + kSmallThreads - 1) / kSmallThreads), (unsigned)p.nsub);
  k_reduce_chunks<<<grid, kSmallThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_eig_polar(const DevPlan& p, int init, cudaStream_t s) {
  if (ns_polar_supported((int)p.kp)) return launch_ns_polar(p, init, s);
  // 80 < kp <= 128: the same fp64 iteration with its matrices in L2 (an fp32
  // iteration carried ~4e-7 into S per iteration, tools/fp32_accuracy.py)
  if (ns_polar_g_supported((int)p.kp) && p.nsg) return launch_ns_polar_g(p, init, s);
  return launch_eig_polar_exact(p, init, s);
}

// fp64 polar transform for every K (NS on DMMA up to kp = 128, Jacobi above)
cudaError_t launch_eig_polar_exact(const DevPlan& p, int init, cudaStream_t s) {
  if (ns_polar_supported((int)p.kp)) return launch_ns_polar(p, init, s);
  if (ns_polar_g_supported((int)p.kp) && p.nsg) return launch_ns_polar_g(p, init, s);
  const size_t bytes = eig_smem_bytes((int)p.K);
  cudaError_t e = set_smem((const void*)k_eig_polar, bytes);
  if (e != cudaSuccess) return e;
  k_eig_polar<<<p.nsub, kSmallThreads, bytes, s>>>(p, init);
  return cudaGetLastError();
}

// the returned W's exact fp64 transform after a fit: fp64 Newton-Schulz up to
// kp = 80; above, where the iterations ran the fp32 Newton-Schulz, its M refined
// in fp64 (k_ns_refine) with Jacobi only for subjects the refinement leaves
cudaError_t launch_final_polar(const DevPlan& p, cudaStream_t s) { return launch_eig_polar_exact(p, 1, s); }

cudaError_t launch_apply_m(const DevPlan& p, int with_cross, cudaStream_t s) {
  const int64_t K4 = (p.K + 3) & ~3;
  const int64_t ldm = p.kp + ((4 - p.kp) % 16 + 16) % 16;
  const size_t bytes = (size_t)(K4 * ldm + K4 * (p.apply_cols + 4)) * sizeof(double);
  const void* fn = nullptr;
  switch (p.kp / 8) {
#define SRM_APPLY_M_CASE(n) \
  case n:                   \
    fn = (const void*)k_apply_m<n, 128>; \
    break;
    SRM_APPLY_M_CASE(1) SRM_APPLY_M_CASE(2) SRM_APPLY_M_CASE(3) SRM_APPLY_M_CASE(4) SRM_APPLY_M_CASE(5)
    SRM_APPLY_M_CASE(6) SRM_APPLY_M_CASE(7) SRM_APPLY_M_CASE(8) SRM_APPLY_M_CASE(9) SRM_APPLY_M_CASE(10)
    SRM_APPLY_M_CASE(11) SRM_APPLY_M_CASE(12) SRM_APPLY_M_CASE(13) SRM_APPLY_M_CASE(14)
#undef SRM_APPLY_M_CASE
    // kp > 112: 64-column tiles (M and the B tile in shared memory: 205 KB at kp = 128)
    case 15: fn = (const void*)k_apply_m<15, 64>; break;
    case 16: fn = (const void*)k_apply_m<16, 64>; break;
    default:
      return cudaErrorInvalidValue;
  }
  if ((p.kp > 112) != (p.apply_cols == 64)) return cudaErrorInvalidValue;
  cudaError_t e = set_smem(fn, bytes);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)p.ntile_apply, (unsigned)p.nsub);
  DevPlan arg = p;
  void* args[] = {&arg, &with_cross};
  e = cudaLaunchKernel(fn, grid, dim3(kSmallThreads), args, bytes, s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_gram_from_b(const DevPlan& p, cudaStream_t s) {
  const size_t bytes = (size_t)2 * p.kp * kGfbLd * sizeof(double);
  const void* fn = nullptr;
  switch (p.kp / 8) {
#define SRM_GFB_CASE(n) \
  case n:               \
    fn = (const void*)k_gram_from_b<8 * n>; \
    break;
    SRM_GFB_CASE(1) SRM_GFB_CASE(2) SRM_GFB_CASE(3) SRM_GFB_CASE(4) SRM_GFB_CASE(5) SRM_GFB_CASE(6)
    SRM_GFB_CASE(7) SRM_GFB_CASE(8) SRM_GFB_CASE(9) SRM_GFB_CASE(10) SRM_GFB_CASE(11) SRM_GFB_CASE(12)
    SRM_GFB_CASE(13) SRM_GFB_CASE(14) SRM_GFB_CASE(15) SRM_GFB_CASE(16)
#undef SRM_GFB_CASE
    default:
      return cudaErrorInvalidValue;
  }
  cudaError_t e = set_smem(fn, bytes);
  if (e != cudaSuccess) return e;
  DevPlan arg = p;
  void* args[] = {&arg};
  if (p.nsub == 0) return cudaSuccess;
  e = cudaLaunchKernel(fn, dim3((unsigned)p.gfb_chunks, (unsigned)p.nsub), dim3(kSmallThreads), args, bytes, s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_finalize_rho(const DevPlan& p, int init, cudaStream_t s) {
  k_finalize_rho<<<(p.nsub + 127) / 128, 128, 0, s>>>(p, init, 0);
  return cudaGetLastError();
}

bool finalize_rho_advances(const DevPlan& p) { return p.nsub <= 1024; }

cudaError_t launch_finalize_rho_advance(const DevPlan& p, cudaStream_t s) {
  if (!finalize_rho_advances(p)) return cudaErrorInvalidValue;
  k_finalize_rho<<<1, (p.nsub + 31) / 32 * 32, 0, s>>>(p, 0, 1);
  return cudaGetLastError();
}

cudaError_t launch_set_iteration(const DevPlan& p, int iteration, int advance, cudaStream_t s) {
  k_set_iteration<<<1, 1, 0, s>>>(p, iteration, advance);
  return cudaGetLastError();
}

cudaError_t launch_reduce_terms(const DevPlan& p, double* dst, const int32_t* order, int count,
                                cudaStream_t s, bool ident) {
  const int64_t n = p.kp * p.ldx;
  // ident: order[j] == j (one rank, or equal shards): no dependent index load
  k_reduce_terms<<<(unsigned)((n + kSmallThreads - 1) / kSmallThreads), kSmallThreads, 0, s>>>(
      p, dst, order, count, ident ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_xchg_pack(const DevPlan& p, cudaStream_t s) {
  if (p.n_local == 0) return cudaSuccess;
  const dim3 grid((unsigned)((p.xrec + kSmallThreads - 1) / kSmallThreads), (unsigned)p.n_local, (unsigned)p.world);
  k_xchg_pack<<<grid, kSmallThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_xchg_reduce(const DevPlan& p, cudaStream_t s) {
  const int64_t kx = p.kp * p.xw;
  k_xchg_reduce<<<(unsigned)((kx + kSmallThreads - 1) / kSmallThreads), kSmallThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_xchg_unpack(const DevPlan& p, cudaStream_t s) {
  const dim3 grid((unsigned)((p.xred + kSmallThreads - 1) / kSmallThreads), (unsigned)p.world);
  k_xchg_unpack<<<grid, kSmallThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tail_inv(const DevPlan& p, cudaStream_t s) {
  switch ((p.K + 15) / 16) {
#define SRM_SWEEP_CASE(r) \
  case r:                 \
    k_tail_inv<r><<<1, kSmallThreads, 0, s>>>(p); \
    break;
    SRM_SWEEP_CASE(1) SRM_SWEEP_CASE(2) SRM_SWEEP_CASE(3) SRM_SWEEP_CASE(4)
    SRM_SWEEP_CASE(5) SRM_SWEEP_CASE(6) SRM_SWEEP_CASE(7)
    default: k_tail_inv<8><<<1, kSmallThreads, 0, s>>>(p); break;
#undef SRM_SWEEP_CASE
  }
  return cudaGetLastError();
}

cudaError_t launch_tail_kk(const DevPlan& p, cudaStream_t s) {
  switch ((p.K + 15) / 16) {
#define SRM_SWEEP_CASE(r) \
  case r:                 \
    k_tail_kk<r><<<1, kSmallThreads, 0, s>>>(p); \
    break;
    SRM_SWEEP_CASE(1) SRM_SWEEP_CASE(2) SRM_SWEEP_CASE(3) SRM_SWEEP_CASE(4)
    SRM_SWEEP_CASE(5) SRM_SWEEP_CASE(6) SRM_SWEEP_CASE(7)
    default: k_tail_kk<8><<<1, kSmallThreads, 0, s>>>(p); break;
#undef SRM_SWEEP_CASE
  }
  return cudaGetLastError();
}

cudaError_t launch_tail_s(const DevPlan& p, cudaStream_t s) {
  const size_t b2 = (size_t)3 * p.K * 33 * sizeof(double);
  cudaError_t e = set_smem((const void*)k_tail_s, b2);
  if (e != cudaSuccess) return e;
  k_tail_s<<<p.ntile_tail, kTailSThreads, b2, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tail_sigma(const DevPlan& p, cudaStream_t s) {
  const size_t b3 = (size_t)(p.K * p.K + 4 * p.ntile_tail) * sizeof(double);
  cudaError_t e = set_smem((const void*)k_tail_sigma, b3);
  if (e != cudaSuccess) return e;
  k_tail_sigma<<<1, kSigmaThreads, b3, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tail(const DevPlan& p, cudaStream_t s) {
  cudaError_t e = launch_tail_inv(p, s);
  if (e == cudaSuccess) e = launch_tail_kk(p, s);
  if (e == cudaSuccess) e = launch_tail_s(p, s);
  if (e == cudaSuccess) e = launch_tail_sigma(p, s);
  return e;
}

cudaError_t launch_mirror_gram(const DevPlan& p, int first, int count, cudaStream_t s) {
  const dim3 grid(256, (unsigned)count);
  k_mirror_gram<<<grid, kSmallThreads, 0, s>>>(p, first);
  return cudaGetLastError();
}

cudaError_t launch_reset(const DevPlan& p, cudaStream_t s) {
  k_reset<<<1, kSmallThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_apply_w(const DevPlan& p, const void* items_a, int n_items, cudaStream_t s) {
  const size_t bytes = (size_t)p.K * p.K * sizeof(double);
  cudaError_t e = set_smem((const void*)k_apply_w, bytes);
  if (e != cudaSuccess) return e;
  if (n_items == 0) return cudaSuccess;
  k_apply_w<<<n_items, kSmallThreads, bytes, s>>>(p, static_cast<const ItemA*>(items_a));
  return cudaGetLastError();
}

cudaError_t launch_apply_w_f32(const DevPlan& p, const void* items_a, int n_items, cudaStream_t s) {
  const size_t bytes = (size_t)p.K * p.K * sizeof(double);
  cudaError_t e = set_smem((const void*)k_apply_w_f32, bytes);
  if (e != cudaSuccess) return e;
  if (n_items == 0) return cudaSuccess;
  k_apply_w_f32<<<n_items, kSmallThreads, bytes, s>>>(p, static_cast<const ItemA*>(items_a));
  return cudaGetLastError();
}

cudaError_t launch_spd_inverse(double* a, int n, int32_t* status, cudaStream_t s) {
  // one instantiation per register block (R = ceil(n / 16)): each gets its
  // own register allocation
  switch ((n + 15) / 16) {
#define SRM_SWEEP_CASE(r) \
  case r:                 \
    k_spd_inverse<r><<<1, kSmallThreads, 0, s>>>(a, n, status); \
    break;
    SRM_SWEEP_CASE(1) SRM_SWEEP_CASE(2) SRM_SWEEP_CASE(3) SRM_SWEEP_CASE(4)
    SRM_SWEEP_CASE(5) SRM_SWEEP_CASE(6) SRM_SWEEP_CASE(7)
    default: k_spd_inverse<8><<<1, kSmallThreads, 0, s>>>(a, n, status); break;
#undef SRM_SWEEP_CASE
  }
  return cudaGetLastError();
}

cudaError_t launch_polar_small(const double* gram, int64_t ldg, int n, double* m, int64_t ldm,
                               int32_t* status, cudaStream_t s) {
  const size_t bytes = eig_smem_bytes(n);
  cudaError_t e = set_smem((const void*)k_polar_small, bytes);
  if (e != cudaSuccess) return e;
  k_polar_small<<<1, kSmallThreads, bytes, s>>>(gram, ldg, n, m, ldm, status);
  return cudaGetLastError();
}

cudaError_t launch_apply_right(const double* a, int64_t lda, int64_t v, int k, const double* m,
                               int64_t ldm, double* w, int64_t ldw, cudaStream_t s) {
  const size_t bytes = (size_t)k * k * sizeof(double);
  cudaError_t e = set_smem((const void*)k_apply_right, bytes);
  if (e != cudaSuccess) return e;
  if (v == 0) return cudaSuccess;
  k_apply_right<<<(unsigned)((v + 63) / 64), kSmallThreads, bytes, s>>>(a, lda, v, k, m, ldm, w, ldw);
  return cudaGetLastError();
}

}  // namespace srm
