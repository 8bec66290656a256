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
//   tail            srm.py:121-142: two Cholesky inverses (kernels.py:168-187),
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
constexpr int kMaxK = 112;

__device__ __forceinline__ double* rec_ptr(const DevPlan& p, int slot) {
  return p.terms + (int64_t)slot * p.term_stride;
}

__device__ __forceinline__ bool failed(const DevPlan& p) { return p.status[0] != 0; }

// ---------------------------------------------------------------------------
// prep: one warp per voxel row
// ---------------------------------------------------------------------------
template <typename TIN, typename TOUT>
__global__ void __launch_bounds__(kSmallThreads) k_prep(DevPlan p, int local, const TIN* __restrict__ x,
                                                        int64_t ld) {
  const int64_t* sj = p.subj + (int64_t)local * kSubjCols;
  const int64_t row0 = sj[SC_ROW_OFF];
  const int64_t V = sj[SC_V];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (kSmallThreads / 32) + warp;
  if (row >= V) return;
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
    out[t] = static_cast<TOUT>(v);
  }
  sq = warp_sum(sq);
  if (lane == 0) {
    p.mu[row0 + row] = mean;
    p.rowsq[row0 + row] = sq;
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
  const int i = blockIdx.y;
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

// Shared tail of the polar factor: rank check on the Gram eigenvalues and
// M = Q diag(lambda^-1/2) Q^T written to global (ldm, zero-padded to mp).
// Returns true when the Gram matrix is numerically rank deficient
// (kernels.py:202-206 raises RankError when s_min < 1e-12 s_max, i.e.
// lambda_min < 1e-24 lambda_max; the Gram route cannot resolve ratios below
// ~1e-16, so a non-positive lambda_min is also rank deficient).
__device__ bool polar_from_eig(const double* C, const double* Q, int n, int ld, double* wsh,
                               double* M, int64_t ldm, int mp) {
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
    s_bad = (nan || !(lmax > 0.0) || !(lmin > 1e-24 * lmax)) ? 1 : 0;
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

__global__ void __launch_bounds__(kSmallThreads) k_eig_polar(DevPlan p, int init) {
  const int iteration = init ? -1 : *p.iter;
  const int cold = (init || iteration == 0) ? 1 : 0;
  extern __shared__ __align__(16) double sm[];
  const int i = blockIdx.x;
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
  const bool bad = polar_from_eig(C, Q, n, ld, wsh, p.mmat + (int64_t)i * kp * kp, kp, kp);
  for (int e = tid; e < kp * kp; e += blockDim.x) {
    const int a = e / kp, b = e - a * kp;
    Qg[e] = (a < n && b < n) ? Q[a * ld + b] : 0.0;
  }
  if (bad && tid == 0) {
    const int64_t* sj = p.subj + (int64_t)i * kSubjCols;
    raise_status(p.status, SRM_ERR_RANK, (int)sj[SC_GLOBAL], iteration);
  }
}

// ---------------------------------------------------------------------------
// apply_m: P_i = M_i^T B_i written into the subject's term record, plus the
// per-tile cross term sum_{f,t} P[f][t] S[f][t]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads) k_apply_m(DevPlan p, int with_cross) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double scratch[32];
  const int tile = blockIdx.x, i = blockIdx.y;
  const int kp = (int)p.kp, K = (int)p.K;
  const int64_t t0 = (int64_t)tile * 64;
  double* Ms = sm;            // [K][K]
  double* Bs = Ms + K * K;    // [K][64]
  const double* Mg = p.mmat + (int64_t)i * kp * kp;
  const double* Bg = p.bred + (int64_t)i * p.kp * p.ldo;
  const int tid = threadIdx.x;
  for (int e = tid; e < K * K; e += blockDim.x) Ms[e] = Mg[(e / K) * kp + (e % K)];
  for (int e = tid; e < K * 64; e += blockDim.x) {
    const int c = e >> 6, t = e & 63;
    Bs[e] = (t0 + t < p.ldx) ? Bg[(int64_t)c * p.ldo + t0 + t] : 0.0;
  }
  __syncthreads();
  const int64_t* sj = p.subj + (int64_t)i * kSubjCols;
  double* P = rec_ptr(p, (int)sj[SC_SLOT]);
  const int t = tid & 63;
  double cross = 0.0;
  if (t0 + t < p.ldx) {
    for (int f = tid >> 6; f < kp; f += kSmallThreads / 64) {
      double v = 0.0;
      if (f < K) {
        for (int c = 0; c < K; ++c) v += Ms[c * K + f] * Bs[c * 64 + t];
        if (with_cross) cross += v * p.S[(int64_t)f * p.ldx + t0 + t];
      }
      P[(int64_t)f * p.ldx + t0 + t] = v;
    }
  }
  if (with_cross) {
    cross = block_sum<kSmallThreads>(cross, scratch);
    if (tid == 0) p.crossp[(int64_t)i * p.ntile_apply + tile] = cross;
  }
}

__device__ __forceinline__ int64_t hist_row(const DevPlan& p, int it) { return (int64_t)(it % p.n_hist) * p.hist_stride; }

__global__ void k_set_iteration(DevPlan p, int iteration, int advance) {
  if (advance) *p.iter += 1;
  else *p.iter = iteration;
}

__global__ void k_finalize_rho(DevPlan p, int init) {
  const int iteration = init ? -1 : *p.iter;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_local) return;
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
                                                                int count) {
  const int64_t n = p.kp * p.ldx;
  const int64_t e = (int64_t)blockIdx.x * kSmallThreads + threadIdx.x;
  if (e < n) {
    double acc = 0.0;
    for (int j = 0; j < count; ++j) {
      const double* rec = rec_ptr(p, order[j]);
      const double v = rec[e] / rec[n + RC_RHO2];
      acc = (j == 0) ? v : acc + v;
    }
    dst[e] = acc;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double rho0 = 0.0, vlog = 0.0, sq = 0.0, vsum = 0.0;
    for (int j = 0; j < count; ++j) {
      const double* rec = rec_ptr(p, order[j]) + n;
      const double r = rec[RC_RHO2];
      rho0 = (j == 0) ? 1.0 / r : rho0 + 1.0 / r;
      vlog += rec[RC_V] * log(r);
      sq += rec[RC_SQNORM] / r;
      vsum += rec[RC_V];
    }
    dst[n + RD_RHO0] = rho0;
    dst[n + RD_VLOGRHO] = vlog;
    dst[n + RD_SQRHO] = sq;
    dst[n + RD_VSUM] = vsum;
  }
}

// ---------------------------------------------------------------------------
// K x K Cholesky helpers (one CTA, matrices in shared memory)
// ---------------------------------------------------------------------------
// In-place lower Cholesky.  Returns -1 on success or the failing 0-based
// pivot (dpotrf info - 1).  *logdet = 2 sum log L_jj.
__device__ int chol_lower(double* A, int n, int ld, double* logdet) {
  __shared__ double s_ljj;
  __shared__ int s_fail;
  const int tid = threadIdx.x;
  double ld_acc = 0.0;
  for (int j = 0; j < n; ++j) {
    __syncthreads();
    if (tid == 0) {
      const double d = A[j * ld + j];
      s_fail = (d > 0.0) ? -1 : j;
      s_ljj = (d > 0.0) ? sqrt(d) : 0.0;
      if (d > 0.0) A[j * ld + j] = s_ljj;
    }
    __syncthreads();
    if (s_fail >= 0) return s_fail;
    const double ljj = s_ljj;
    ld_acc += log(ljj);
    for (int r = j + 1 + tid; r < n; r += blockDim.x) A[r * ld + j] /= ljj;
    __syncthreads();
    const int m = n - j - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int r = j + 1 + e / m, c = j + 1 + e % m;
      if (c <= r) A[r * ld + c] -= A[r * ld + j] * A[c * ld + j];
    }
  }
  __syncthreads();
  *logdet = 2.0 * ld_acc;
  return -1;
}

// Linv (lower) = inverse of lower-triangular L; one thread per column.
__device__ void tri_inverse(const double* L, double* Li, int n, int ld) {
  const int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += blockDim.x) Li[(e / n) * ld + (e % n)] = 0.0;
  __syncthreads();
  for (int c = tid; c < n; c += blockDim.x) {
    Li[c * ld + c] = 1.0 / L[c * ld + c];
    for (int r = c + 1; r < n; ++r) {
      double s = 0.0;
      for (int k = c; k < r; ++k) s += L[r * ld + k] * Li[k * ld + c];
      Li[r * ld + c] = -s / L[r * ld + r];
    }
  }
  __syncthreads();
}

// A = Li^T Li (symmetric, lower computed then mirrored: dpotri + symmetrise)
__device__ void gram_lower(const double* Li, double* A, int n, int ld) {
  const int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int a = e / n, b = e - a * n;
    if (a >= b) {
      double s = 0.0;
      for (int k = a; k < n; ++k) s += Li[k * ld + a] * Li[k * ld + b];
      A[a * ld + b] = s;
    }
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int a = e / n, b = e - a * n;
    if (a < b) A[a * ld + b] = A[b * ld + a];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// tail, stage 1 (one CTA): var_s and C = Sigma_s^T (I - rho0 var_s)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads) k_tail_kk(DevPlan p) {
  const int iteration = *p.iter;
  extern __shared__ __align__(16) double sm[];
  if (failed(p)) return;
  const int n = (int)p.K, ld = n + 1, kp = (int)p.kp;
  double* M1 = sm;
  double* M2 = sm + n * ld;
  const int tid = threadIdx.x;
  const double rho0 = p.red[p.kp * p.ldx + RD_RHO0];
  for (int e = tid; e < n * n; e += blockDim.x) M1[(e / n) * ld + e % n] = p.sigma[(e / n) * kp + e % n];
  double logdet_sigma = 0.0, logdet_prec = 0.0;
  int piv = chol_lower(M1, n, ld, &logdet_sigma);
  if (piv >= 0) {
    if (tid == 0) raise_status(p.status, SRM_ERR_DEFINITENESS, piv, iteration);
    return;
  }
  tri_inverse(M1, M2, n, ld);
  gram_lower(M2, M1, n, ld);  // Sigma_s^{-1}
  for (int j = tid; j < n; j += blockDim.x) M1[j * ld + j] += rho0;
  piv = chol_lower(M1, n, ld, &logdet_prec);
  if (piv >= 0) {
    if (tid == 0) raise_status(p.status, SRM_ERR_DEFINITENESS, piv, iteration);
    return;
  }
  tri_inverse(M1, M2, n, ld);
  gram_lower(M2, M1, n, ld);  // var_s
  for (int e = tid; e < kp * kp; e += blockDim.x) {
    const int a = e / kp, b = e - a * kp;
    p.var[e] = (a < n && b < n) ? M1[a * ld + b] : 0.0;
  }
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int a = e / n, b = e - a * n;
    M2[a * ld + b] = (a == b ? 1.0 : 0.0) - rho0 * M1[a * ld + b];
  }
  __syncthreads();
  for (int e = tid; e < kp * kp; e += blockDim.x) {
    const int a = e / kp, b = e - a * kp;
    double s = 0.0;
    if (a < n && b < n)
      for (int k = 0; k < n; ++k) s += p.sigma[k * kp + a] * M2[k * ld + b];
    p.cmat[e] = s;
  }
  if (tid == 0) {
    p.tailscr[TS_LOGDET_SIGMA] = logdet_sigma;
    p.tailscr[TS_LOGDET_PREC] = logdet_prec;
  }
}

// tail, stage 2 (32-column tiles): S = C red, quad = <red, var red>, S S^T
// partials and the tolerance statistics.
__global__ void __launch_bounds__(kSmallThreads) k_tail_s(DevPlan p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double scratch[32];
  if (failed(p)) return;
  const int K = (int)p.K, kp = (int)p.kp;
  const int tile = blockIdx.x;
  const int64_t t0 = (int64_t)tile * 32;
  double* Rt = sm;           // [K][32]
  double* St = sm + K * 32;  // [K][32]
  const int tid = threadIdx.x, col = tid & 31, rg = tid >> 5;
  const int64_t t = t0 + col;
  const bool tin = t < p.ldx;
  for (int f = rg; f < K; f += 8) Rt[f * 32 + col] = tin ? p.red[(int64_t)f * p.ldx + t] : 0.0;
  __syncthreads();
  double quad = 0.0, dsq = 0.0, osq = 0.0;
  for (int f = rg; f < K; f += 8) {
    double s = 0.0, y = 0.0;
    for (int c = 0; c < K; ++c) {
      const double r = Rt[c * 32 + col];
      s += p.cmat[f * kp + c] * r;
      y += p.var[f * kp + c] * r;
    }
    quad += Rt[f * 32 + col] * y;
    St[f * 32 + col] = s;
    if (tin && p.st) p.st[t * kp + f] = s;
    if (tin && p.sf) {
      const float sfv = (float)s;
      const float hi = __uint_as_float(__float_as_uint(sfv) & 0xFFFFE000u);
      p.sf[(int64_t)f * p.ldx + t] = hi;
      p.sf[(int64_t)(p.np + f) * p.ldx + t] = sfv - hi;
    }
    if (tin) {
      double* sp = p.S + (int64_t)f * p.ldx + t;
      const double old = *sp;
      dsq += (s - old) * (s - old);
      osq += old * old;
      *sp = s;
    }
  }
  __syncthreads();
  double* ssp = p.sspart + (int64_t)tile * kp * kp;
  for (int e = tid; e < K * K; e += blockDim.x) {
    const int a = e / K, b = e - a * K;
    double v = 0.0;
#pragma unroll 8
    for (int c = 0; c < 32; ++c) v += St[a * 32 + c] * St[b * 32 + c];
    ssp[a * kp + b] = v;
  }
  quad = block_sum<kSmallThreads>(quad, scratch);
  dsq = block_sum<kSmallThreads>(dsq, scratch);
  osq = block_sum<kSmallThreads>(osq, scratch);
  if (tid == 0) {
    p.tailpart[tile * 4 + 0] = quad;
    p.tailpart[tile * 4 + 1] = dsq;
    p.tailpart[tile * 4 + 2] = osq;
  }
}

// tail, stage 3 (one CTA): Sigma_s <- sym(var_s + S S^T / T), trace, LL
__global__ void __launch_bounds__(kSmallThreads) k_tail_sigma(DevPlan p) {
  const int iteration = *p.iter;
  extern __shared__ __align__(16) double sm[];
  if (failed(p)) return;
  const int K = (int)p.K, kp = (int)p.kp;
  const int tid = threadIdx.x;
  const double T = (double)p.T;
  double* Sn = sm;  // [K][K]
  for (int e = tid; e < K * K; e += blockDim.x) {
    const int a = e / K, b = e - a * K;
    double ss = 0.0;
    for (int tile = 0; tile < p.ntile_tail; ++tile) ss += p.sspart[(int64_t)tile * kp * kp + a * kp + b];
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
    for (int tile = 0; tile < p.ntile_tail; ++tile) {
      quad += p.tailpart[tile * 4 + 0];
      dsq += p.tailpart[tile * 4 + 1];
      osq += p.tailpart[tile * 4 + 2];
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
  }
  if (threadIdx.x == 0) {
    p.status[0] = p.status[1] = p.status[2] = 0;
    *p.iter = 0;
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
__global__ void __launch_bounds__(kSmallThreads) k_spd_inverse(double* a, int n, int32_t* status) {
  extern __shared__ __align__(16) double sm[];
  const int ld = n + 1;
  double* M1 = sm;
  double* M2 = sm + n * ld;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) M1[(e / n) * ld + e % n] = a[e];
  double logdet;
  const int piv = chol_lower(M1, n, ld, &logdet);
  if (piv >= 0) {
    if (threadIdx.x == 0) raise_status(status, SRM_ERR_DEFINITENESS, piv, -1);
    return;
  }
  tri_inverse(M1, M2, n, ld);
  gram_lower(M2, M1, n, ld);
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) a[e] = M1[(e / n) * ld + e % n];
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
  const bool bad = polar_from_eig(C, Q, n, ld, wsh, m, ldm, n);
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
cudaError_t set_smem(const void* f, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static const void* funcs[32];
  static size_t limits[32];
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
  if (e == cudaSuccess && n < 32) {
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
  const dim3 grid((unsigned)((V + 7) / 8));
  if (V == 0) return cudaSuccess;
  if (x_dtype == SRM_F64 && xhat_dtype == SRM_F64)
    k_prep<double, double><<<grid, kSmallThreads, 0, s>>>(p, local, static_cast<const double*>(x), ld);
  else if (x_dtype == SRM_F64 && xhat_dtype == SRM_F32)
    k_prep<double, float><<<grid, kSmallThreads, 0, s>>>(p, local, static_cast<const double*>(x), ld);
  else if (x_dtype == SRM_F32 && xhat_dtype == SRM_F32)
    k_prep<float, float><<<grid, kSmallThreads, 0, s>>>(p, local, static_cast<const float*>(x), ld);
  else
    k_prep<float, double><<<grid, kSmallThreads, 0, s>>>(p, local, static_cast<const float*>(x), ld);
  return cudaGetLastError();
}

cudaError_t launch_subject_sqnorm(const DevPlan& p, cudaStream_t s) {
  k_subject_sqnorm<<<p.n_local, kSmallThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_reduce_chunks(const DevPlan& p, cudaStream_t s) {
  const int64_t n2 = p.kp * p.ldo / 2;
  const dim3 grid((unsigned)((n2 + kSmallThreads - 1) / kSmallThreads), (unsigned)p.n_local);
  k_reduce_chunks<<<grid, kSmallThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_eig_polar(const DevPlan& p, int init, cudaStream_t s) {
  if (ns_polar_supported((int)p.kp)) return launch_ns_polar(p, init, s);
  if ((p.flags & SRM_FLAG_TC) && ns_polar_f32_supported((int)p.kp)) return launch_ns_polar_f32(p, init, s);
  return launch_eig_polar_exact(p, init, s);
}

// fp64 polar transform for every K (NS on DMMA up to kp = 80, Jacobi above)
cudaError_t launch_eig_polar_exact(const DevPlan& p, int init, cudaStream_t s) {
  if (ns_polar_supported((int)p.kp)) return launch_ns_polar(p, init, s);
  const size_t bytes = eig_smem_bytes((int)p.K);
  cudaError_t e = set_smem((const void*)k_eig_polar, bytes);
  if (e != cudaSuccess) return e;
  k_eig_polar<<<p.n_local, kSmallThreads, bytes, s>>>(p, init);
  return cudaGetLastError();
}

cudaError_t launch_apply_m(const DevPlan& p, int with_cross, cudaStream_t s) {
  const size_t bytes = (size_t)(p.K * p.K + p.K * 64) * sizeof(double);
  cudaError_t e = set_smem((const void*)k_apply_m, bytes);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)p.ntile_apply, (unsigned)p.n_local);
  k_apply_m<<<grid, kSmallThreads, bytes, s>>>(p, with_cross);
  return cudaGetLastError();
}

cudaError_t launch_finalize_rho(const DevPlan& p, int init, cudaStream_t s) {
  k_finalize_rho<<<(p.n_local + 127) / 128, 128, 0, s>>>(p, init);
  return cudaGetLastError();
}

cudaError_t launch_set_iteration(const DevPlan& p, int iteration, int advance, cudaStream_t s) {
  k_set_iteration<<<1, 1, 0, s>>>(p, iteration, advance);
  return cudaGetLastError();
}

cudaError_t launch_reduce_terms(const DevPlan& p, double* dst, const int32_t* order, int count,
                                cudaStream_t s) {
  const int64_t n = p.kp * p.ldx;
  k_reduce_terms<<<(unsigned)((n + kSmallThreads - 1) / kSmallThreads), kSmallThreads, 0, s>>>(
      p, dst, order, count);
  return cudaGetLastError();
}

cudaError_t launch_tail_kk(const DevPlan& p, cudaStream_t s) {
  const int K = (int)p.K;
  const size_t b1 = (size_t)2 * K * (K + 1) * sizeof(double);
  cudaError_t e = set_smem((const void*)k_tail_kk, b1);
  if (e != cudaSuccess) return e;
  k_tail_kk<<<1, kSmallThreads, b1, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tail_s(const DevPlan& p, cudaStream_t s) {
  const size_t b2 = (size_t)2 * p.K * 32 * sizeof(double);
  cudaError_t e = set_smem((const void*)k_tail_s, b2);
  if (e != cudaSuccess) return e;
  k_tail_s<<<p.ntile_tail, kSmallThreads, b2, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tail_sigma(const DevPlan& p, cudaStream_t s) {
  const size_t b3 = (size_t)p.K * p.K * sizeof(double);
  cudaError_t e = set_smem((const void*)k_tail_sigma, b3);
  if (e != cudaSuccess) return e;
  k_tail_sigma<<<1, kSmallThreads, b3, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_tail(const DevPlan& p, cudaStream_t s) {
  cudaError_t e = launch_tail_kk(p, s);
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
  const size_t bytes = (size_t)2 * n * (n + 1) * sizeof(double);
  cudaError_t e = set_smem((const void*)k_spd_inverse, bytes);
  if (e != cudaSuccess) return e;
  k_spd_inverse<<<1, kSmallThreads, bytes, s>>>(a, n, status);
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
