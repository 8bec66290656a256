// Accurate polar transform of a tall V x K matrix A (kernels.py:190-212):
// Householder TSQR for R (A = Q R), then a one-sided Jacobi SVD of the K x K
// R = U_R diag(sigma) V^T, then M = V diag(1/sigma) V^T so that W = A M is the
// polar factor U_R V^T of A's own SVD.
//
// The Gram route of the fit (M = (A^T A)^{-1/2} from A^T A, polar_ns.cu /
// smallmat.cu) squares cond(A): its small eigenvalues carry an absolute error
// of ~eps |A|^2, so sigma_min / sigma_max below ~1e-8 cannot be resolved.  This
// route never forms A^T A: Householder QR is backward stable and one-sided
// Jacobi resolves the singular values of R to ~eps sigma_max, like the
// reference's gesdd, so the rank test sigma_min < 1e-12 sigma_max
// (kernels.py:202-206) is decided exactly as the reference decides it.
//
// TSQR: level 0 splits every matrix into row ranges, one CTA per range; each
// CTA streams its range in blocks of B rows and keeps R_acc (K x K) in shared
// memory, factoring [R_acc; block] with K Householder reflectors that each
// touch one row of R_acc and the B block rows (the triangle below the
// diagonal of R_acc is zero).  Level L > 0 runs the same kernel on the
// stacked K x K factors of level L - 1 until one R per matrix remains.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace srm {

namespace {

constexpr int kQrThreads = 512;
constexpr int kSvdThreads = 512;

__global__ void __launch_bounds__(kQrThreads) k_tsqr(const QrJob* __restrict__ jobs, int K, int B) {
  extern __shared__ __align__(16) double qsm[];
  __shared__ double s_par[2];
  const QrJob jb = jobs[blockIdx.y];
  const int c = blockIdx.x;
  if (c >= jb.nctas) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kQrThreads / 32;
  const int LD = K + 1;  // odd pitch: a warp walking a column hits every bank pair twice
  double* M = qsm;       // rows 0..K-1: R_acc; rows K..K+B-1: the block
  for (int e = tid; e < K * LD; e += kQrThreads) M[e] = 0.0;
  const int64_t r_begin = (int64_t)c * jb.rpc;
  const int64_t r_end = min(jb.rows, r_begin + jb.rpc);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += B) {
    const int nb = (int)min((int64_t)B, r_end - r0);
    __syncthreads();  // the previous block's updates are complete
    for (int e = tid; e < nb * K; e += kQrThreads) {
      const int r = e / K, col = e - r * K;
      M[(K + r) * LD + col] = jb.a[(r0 + r) * jb.lda + col];
    }
    __syncthreads();
    for (int j = 0; j < K; ++j) {
      if (warp == 0) {
        double s = 0.0;
        for (int r = lane; r < nb; r += 32) {
          const double x = M[(K + r) * LD + j];
          s = fma(x, x, s);
        }
        s = warp_sum(s);
        if (lane == 0) {
          const double alpha = M[j * LD + j];
          double tau = 0.0, scale = 0.0;
          if (s > 0.0) {  // dlarfg: beta = -sign(alpha) |x|, v = x / (alpha - beta), v_j = 1
            const double beta = -copysign(sqrt(fma(alpha, alpha, s)), alpha);
            tau = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
            M[j * LD + j] = beta;
          }
          s_par[0] = tau;
          s_par[1] = scale;
        }
      }
      __syncthreads();
      const double tau = s_par[0], scale = s_par[1];
      if (tau != 0.0) {
        for (int col = j + 1 + warp; col < K; col += NW) {
          double d = 0.0;
          for (int r = lane; r < nb; r += 32) d = fma(M[(K + r) * LD + j], M[(K + r) * LD + col], d);
          d = warp_sum(d);
          const double w = tau * fma(scale, d, M[j * LD + col]);  // tau v^T y
          if (lane == 0) M[j * LD + col] -= w;
          const double ws = w * scale;
          for (int r = lane; r < nb; r += 32) M[(K + r) * LD + col] -= ws * M[(K + r) * LD + j];
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  double* out = jb.rout + (int64_t)c * K * K;
  for (int e = tid; e < K * K; e += kQrThreads) {
    const int r = e / K, col = e - r * K;
    out[e] = r <= col ? M[r * LD + col] : 0.0;
  }
}

__device__ __forceinline__ int rr_pair(int i, int r, int np2) { return i == 0 ? 0 : 1 + ((i - 1 + r) % (np2 - 1)); }

// One CTA per job: R (K x K, pitch K) -> M = V diag(1 / sigma) V^T (pitch ldm,
// zero-padded to mp x mp).  Rank test as kernels.py:202-206.
__global__ void __launch_bounds__(kSvdThreads) k_svd_polar(const SvdJob* __restrict__ jobs, int K, int32_t* status,
                                                          const int32_t* iter) {
  extern __shared__ __align__(16) double vsm[];
  __shared__ double s_sig[2];
  const SvdJob jb = jobs[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kSvdThreads / 32;
  const int LD = K + 1;
  // U (R, rotated in place: its columns become U_R sigma) in shared memory; the
  // accumulated rotations V too while both fit (K <= 112), else in the job's
  // global scratch (L2-resident), pitch K
  const bool vsmem = jb.vg == nullptr;
  double* U = vsm;
  double* sig = U + K * LD;                   // column norms
  double* V = vsmem ? sig + K : jb.vg;
  const int LV = vsmem ? LD : K;
  for (int e = tid; e < K * K; e += kSvdThreads) {
    const int r = e / K, col = e - r * K;
    U[r * LD + col] = jb.r[e];
    V[r * LV + col] = r == col ? 1.0 : 0.0;
  }
  __syncthreads();
  const int np2 = (K + 1) & ~1;
  const double tol = fmax(1e-15, sqrt((double)K) * 2.220446049250313e-16);
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rot = 0;
    for (int round = 0; round < np2 - 1; ++round) {
      for (int j = warp; j < np2 / 2; j += NW) {
        const int a = rr_pair(j, round, np2), b = rr_pair(np2 - 1 - j, round, np2);
        const int p = min(a, b), q = max(a, b);
        if (q >= K) continue;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < K; r += 32) {
          const double up = U[r * LD + p], uq = U[r * LD + q];
          al = fma(up, up, al);
          be = fma(uq, uq, be);
          ga = fma(up, uq, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga == 0.0 || !(fabs(ga) > tol * sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double cs = 1.0 / sqrt(fma(t, t, 1.0)), sn = cs * t;
        for (int r = lane; r < K; r += 32) {
          const double up = U[r * LD + p], uq = U[r * LD + q];
          U[r * LD + p] = cs * up - sn * uq;
          U[r * LD + q] = sn * up + cs * uq;
          const double vp = V[r * LV + p], vq = V[r * LV + q];
          V[r * LV + p] = cs * vp - sn * vq;
          V[r * LV + q] = sn * vp + cs * vq;
        }
        rot = 1;
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rot)) break;
  }
  for (int col = warp; col < K; col += NW) {
    double s = 0.0;
    for (int r = lane; r < K; r += 32) s = fma(U[r * LD + col], U[r * LD + col], s);
    s = warp_sum(s);
    if (lane == 0) sig[col] = sqrt(s);
  }
  __syncthreads();
  if (tid == 0) {
    double smax = 0.0, smin = sig[0];
    bool nan = false;
    for (int j = 0; j < K; ++j) {
      nan |= isnan(sig[j]);
      smax = fmax(smax, sig[j]);
      smin = fmin(smin, sig[j]);
    }
    s_sig[0] = smax;
    s_sig[1] = smin;
    // kernels.py:202-206: s[0] == 0 or s[-1] < 1e-12 s[0] raises RankError
    if (nan || !(smax > 0.0) || !(smin >= 1e-12 * smax))
      raise_status(status, SRM_ERR_RANK, jb.subject, iter ? *iter : -1);
  }
  __syncthreads();
  for (int j = tid; j < K; j += kSvdThreads) sig[j] = sig[j] > 0.0 ? 1.0 / sig[j] : 0.0;
  __syncthreads();
  for (int e = tid; e < jb.mp * jb.mp; e += kSvdThreads) {
    const int a = e / jb.mp, b = e - a * jb.mp;
    double m = 0.0;
    if (a < K && b < K)
      for (int j = 0; j < K; ++j) m = fma(V[a * LV + j] * V[b * LV + j], sig[j], m);
    jb.m[(int64_t)a * jb.ldm + b] = m;
  }
}

cudaError_t smem_attr(const void* f, size_t bytes, size_t* cache) {
  if (bytes <= 48 * 1024 || bytes <= *cache) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) *cache = bytes;
  return e;
}

}  // namespace

int tsqr_block_rows(int K) {
  const int fit = (int)((200 * 1024) / (8 * (K + 1))) - K;
  return std::max(32, std::min(256, fit / 32 * 32));
}

bool qr_polar_supported(int K) {
  return K >= 1 && K <= 128 && (size_t)(K + tsqr_block_rows(K)) * (K + 1) * 8 <= 227 * 1024;
}

bool svd_needs_global_v(int K) { return (size_t)(2 * K * (K + 1) + K) * 8 > 227 * 1024; }

TsqrSchedule tsqr_schedule(const std::vector<int64_t>& rows, int K, int target_ctas) {
  TsqrSchedule s;
  const int n = (int)rows.size();
  const int B = tsqr_block_rows(K);
  int64_t total = 0;
  for (int64_t r : rows) total += r;
  std::vector<int64_t> cur = rows;
  bool first = true;
  while (true) {
    std::vector<TsqrSchedule::Job> lvl;
    int64_t acc = 0;
    bool done = true;
    for (int i = 0; i < n; ++i) {
      int64_t rpc;
      if (first) {
        // about target_ctas CTAs over all matrices, at least one block each
        const int64_t share = std::max<int64_t>(1, (int64_t)target_ctas * cur[i] / std::max<int64_t>(total, 1));
        rpc = std::max<int64_t>(B, (cur[i] + share - 1) / share);
      } else {
        rpc = 8 * (int64_t)K;  // eight stacked factors per CTA
      }
      const int nctas = (int)std::max<int64_t>(1, (cur[i] + rpc - 1) / rpc);
      lvl.push_back({cur[i], rpc, nctas, acc});
      acc += (int64_t)nctas * K * K;
      if (nctas > 1) done = false;
    }
    s.levels.push_back(lvl);
    s.buf_doubles = std::max(s.buf_doubles, acc);
    for (int i = 0; i < n; ++i) cur[i] = (int64_t)lvl[i].nctas * K;
    first = false;
    if (done) break;
  }
  return s;
}

std::vector<std::vector<QrJob>> tsqr_jobs(const TsqrSchedule& s, const std::vector<const double*>& a,
                                          const std::vector<int64_t>& lda, int K, double* buf0, double* buf1,
                                          std::vector<const double*>* r_final) {
  std::vector<std::vector<QrJob>> out;
  double* bufs[2] = {buf0, buf1};
  for (size_t L = 0; L < s.levels.size(); ++L) {
    std::vector<QrJob> lvl;
    for (size_t i = 0; i < s.levels[L].size(); ++i) {
      const TsqrSchedule::Job& j = s.levels[L][i];
      QrJob q;
      if (L == 0) {
        q.a = a[i];
        q.lda = lda[i];
      } else {
        q.a = bufs[(L - 1) % 2] + s.levels[L - 1][i].out_off;
        q.lda = K;
      }
      q.rows = j.rows;
      q.rpc = j.rpc;
      q.rout = bufs[L % 2] + j.out_off;
      q.nctas = j.nctas;
      q.pad = 0;
      lvl.push_back(q);
    }
    out.push_back(lvl);
  }
  if (r_final) {
    r_final->clear();
    const size_t L = s.levels.size() - 1;
    for (size_t i = 0; i < s.levels[L].size(); ++i) r_final->push_back(bufs[L % 2] + s.levels[L][i].out_off);
  }
  return out;
}

int tsqr_max_ctas(const std::vector<TsqrSchedule::Job>& lvl) {
  int m = 0;
  for (const auto& j : lvl) m = std::max(m, j.nctas);
  return m;
}

cudaError_t launch_tsqr(const QrJob* jobs_dev, int n_jobs, int max_ctas, int K, cudaStream_t st) {
  static size_t cache = 0;
  const int B = tsqr_block_rows(K);
  const size_t bytes = (size_t)(K + B) * (K + 1) * sizeof(double);
  cudaError_t e = smem_attr((const void*)k_tsqr, bytes, &cache);
  if (e != cudaSuccess || n_jobs == 0 || max_ctas == 0) return e;
  k_tsqr<<<dim3((unsigned)max_ctas, (unsigned)n_jobs), kQrThreads, bytes, st>>>(jobs_dev, K, B);
  return cudaGetLastError();
}

cudaError_t launch_svd_polar(const SvdJob* jobs_dev, int n_jobs, int K, int32_t* status, const int32_t* iter,
                             cudaStream_t st) {
  static size_t cache = 0;
  const size_t bytes = (size_t)((svd_needs_global_v(K) ? 1 : 2) * K * (K + 1) + K) * sizeof(double);
  cudaError_t e = smem_attr((const void*)k_svd_polar, bytes, &cache);
  if (e != cudaSuccess || n_jobs == 0) return e;
  k_svd_polar<<<(unsigned)n_jobs, kSvdThreads, bytes, st>>>(jobs_dev, K, status, iter);
  return cudaGetLastError();
}

}  // namespace srm
