// Stateless step kernels behind the reference's per-step API
// (srm.py:116-155 e_step_local / m_step_subject pieces, kernels.py:168-212).
// They stage their operands into zero-padded workspace copies (so any caller
// layout is accepted) and reuse the same DMMA contraction kernels as the fit.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/srm_b200.h"
#include "common.cuh"
#include "kernels.h"
#include "plan.h"

using namespace srm;

namespace {

inline int64_t rup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
constexpr int64_t kChunk = 2048;

struct Carve {
  char* base;
  int64_t used = 0;
  int64_t cap;
  template <typename T>
  T* take(int64_t n) {
    T* p = reinterpret_cast<T*>(base + used);
    used += rup(n * (int64_t)sizeof(T), 256);
    return used <= cap ? p : nullptr;
  }
};

__global__ void k_sum_chunks(const double* __restrict__ part, int64_t stride, int nch, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= stride) return;
  double acc = part[e];
  for (int c = 1; c < nch; ++c) acc += part[(int64_t)c * stride + e];
  out[e] = acc;
}

// sum of squares of an [rows x cols] block (pitch lda) in a fixed order:
// CTA c takes elements [c per, (c + 1) per) of the row-major enumeration, a
// second single-CTA pass sums the CTA partials; non-finite entries raise
// InvalidInputError (kernels.py:45-46)
constexpr int kSqThreads = 256;

__global__ void __launch_bounds__(kSqThreads) k_sumsq_part(const double* __restrict__ a, int64_t lda, int64_t rows,
                                                          int64_t cols, int64_t per, double* __restrict__ part,
                                                          int32_t* status) {
  __shared__ double scratch[32];
  const int64_t n = rows * cols;
  const int64_t e0 = (int64_t)blockIdx.x * per, e1 = min(n, e0 + per);
  double s = 0.0;
  bool bad = false;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kSqThreads) {
    const int64_t r = e / cols, c = e - r * cols;
    const double x = a[r * lda + c];
    bad |= !isfinite(x);
    s = fma(x, x, s);
  }
  s = block_sum<kSqThreads>(s, scratch);
  if (__syncthreads_or(bad) && threadIdx.x == 0) raise_status(status, SRM_ERR_INVALID_INPUT, 0, -1);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kSqThreads) k_sum_final(const double* __restrict__ part, int n, double* out) {
  __shared__ double scratch[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kSqThreads) s += part[i];
  s = block_sum<kSqThreads>(s, scratch);
  if (threadIdx.x == 0) *out = s;
}

// M = (3 I - G) / 2 for a symmetric G (the Newton-Schulz polar step), symmetrised
__global__ void k_ns_step_matrix(const double* __restrict__ g, int64_t ldg, int n, double* __restrict__ m,
                                 int64_t ldm) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int r = e / n, c = e - r * n;
  const double gs = 0.5 * (g[(int64_t)r * ldg + c] + g[(int64_t)c * ldg + r]);
  m[(int64_t)r * ldm + c] = 0.5 * ((r == c ? 3.0 : 0.0) - gs);
}

cudaError_t launch_ns_step_matrix(const double* g, int64_t ldg, int n, double* m, int64_t ldm, cudaStream_t st) {
  k_ns_step_matrix<<<(n * n + 255) / 256, 256, 0, st>>>(g, ldg, n, m, ldm);
  return cudaGetLastError();
}

// sum_{r,c} a[r][c] b[r][c] in a fixed order (per-CTA partials, then one CTA)
__global__ void __launch_bounds__(kSqThreads) k_dot_part(const double* __restrict__ a, int64_t lda,
                                                        const double* __restrict__ b, int64_t ldb, int64_t rows,
                                                        int64_t cols, int64_t per, double* __restrict__ part) {
  __shared__ double scratch[32];
  const int64_t n = rows * cols;
  const int64_t e0 = (int64_t)blockIdx.x * per, e1 = min(n, e0 + per);
  double s = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kSqThreads) {
    const int64_t r = e / cols, c = e - r * cols;
    s = fma(a[r * lda + c], b[r * ldb + c], s);
  }
  s = block_sum<kSqThreads>(s, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// srm.py:140-142: Sigma_new = sym(var_s + S S^T / T), trace(Sigma_new) (ss = S S^T)
__global__ void __launch_bounds__(kSqThreads) k_sigma_update(const double* __restrict__ var, int64_t ldv,
                                                            const double* __restrict__ ss, int64_t ldss, int n,
                                                            double inv_t, double* __restrict__ out, int64_t ldo,
                                                            double* __restrict__ trace) {
  __shared__ double scratch[32];
  double tr = 0.0;
  for (int e = threadIdx.x; e < n * n; e += kSqThreads) {
    const int r = e / n, c = e - r * n;
    const double nrc = var[(int64_t)r * ldv + c] + ss[(int64_t)r * ldss + c] * inv_t;
    const double ncr = var[(int64_t)c * ldv + r] + ss[(int64_t)c * ldss + r] * inv_t;
    const double v = 0.5 * (nrc + ncr);
    out[(int64_t)r * ldo + c] = v;
    if (r == c) tr += v;
  }
  tr = block_sum<kSqThreads>(tr, scratch);
  if (threadIdx.x == 0) *trace = tr;
}

__global__ void k_add_diag(const double* __restrict__ a, int64_t lda, int64_t n, double c, double* __restrict__ out,
                           int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const int64_t r = e / n, col = e - r * n;
  out[r * ldo + col] = r == col ? a[r * lda + col] + c : a[r * lda + col];
}

int ret(cudaError_t e, const char* where = "stateless") {
  if (e == cudaSuccess) return SRM_OK;
  set_last_error(where, e);
  return SRM_ERR_CUDA;
}

// out (kp x ncols_pad) = L^T R over v rows, L [v x kp] f64, R [v x ldr] dtype
cudaError_t split_v(const double* L, int64_t kp, const void* R, int r_dtype, int64_t ldr, int64_t ncols,
                    int64_t v, double alpha, double* part, double* out, ItemE* items_dev, cudaStream_t st) {
  const int nch = (int)std::max<int64_t>(1, (v + kChunk - 1) / kChunk);
  std::vector<ItemE> items;
  for (int c = 0; c < nch; ++c) {
    const int64_t r0 = (int64_t)c * kChunk;
    for (int64_t n0 = 0; n0 < ncols; n0 += 128) {
      ItemE it;
      it.l_off = r0 * kp;
      it.r_off = r0 * ldr + n0;
      it.o_off = (int64_t)c * kp * ncols + n0;
      it.rows = (int32_t)std::max<int64_t>(0, std::min<int64_t>(kChunk, v - r0));
      it.ncols = (int32_t)std::min<int64_t>(128, ncols - n0);
      it.mrows = (int32_t)kp;
      it.pad = 0;
      items.push_back(it);
    }
  }
  cudaError_t e = cudaMemcpyAsync(items_dev, items.data(), items.size() * sizeof(ItemE), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  e = launch_contract_e((int)kp, SRM_F64, r_dtype, L, kp, R, ldr, part, ncols, alpha, items_dev, (int)items.size(), st);
  if (e != cudaSuccess) return e;
  const int64_t n = kp * ncols;
  k_sum_chunks<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, n, nch, out);
  return cudaGetLastError();
}

constexpr int kPolarCtas = 296;  // level-0 TSQR CTAs: two per SM

int64_t polar_workspace_bytes(int64_t v, int64_t k) {
  if (k < 1 || v < 1) return 0;
  const int64_t kp = rup(k, 8);
  const int64_t nch = std::max<int64_t>(1, (v + kChunk - 1) / kChunk);
  const TsqrSchedule sch = tsqr_schedule({v}, (int)k, kPolarCtas);
  int64_t b = 0;
  b += 2 * rup(v * kp * 8, 256);                              // A copy, W = A M
  b += 2 * rup(sch.buf_doubles * 8, 256);                     // TSQR factors (ping-pong)
  b += rup(nch * kp * kp * 8, 256) + 4 * rup(kp * kp * 8, 256);  // W^T W partials, G, M, M2, SVD V
  b += rup((int64_t)sch.levels.size() * sizeof(QrJob), 256) + rup(sizeof(SvdJob), 256);
  b += rup(nch * (int64_t)sizeof(ItemE), 256);
  return b;
}

}  // namespace

extern "C" {

int64_t srm_stateless_workspace_bytes(int64_t v, int64_t k, int64_t t) {
  const int64_t kp = rup(k, 8), ldxp = rup(t, 32);
  const int64_t nch = std::max<int64_t>(1, (v + kChunk - 1) / kChunk);
  const int64_t ntile = (std::max(ldxp, kp) + 127) / 128;
  int64_t b = 0;
  b += rup(v * kp * 8, 256);                         // L / A copy
  b += rup(v * ldxp * 8, 256);                       // X copy
  b += rup(nch * kp * std::max(ldxp, kp) * 8, 256);  // partials
  b += rup(kp * std::max(ldxp, kp) * 8, 256);        // reduced
  b += rup(v * kp * 8, 256);                         // T-contraction output
  b += rup(kp * kp * 8 * 2, 256);                    // M / scratch
  b += rup(nch * ntile * (int64_t)sizeof(ItemE) + ((v + 127) / 128) * (int64_t)sizeof(ItemA), 256);
  // tail step: red, S (kp x ldx), sigma/var/cmat, per-tile partials
  const int64_t ntail = ldxp / 32;
  b += rup((2 * kp * ldxp + 16) * 8, 256) + rup((4 + ntail) * kp * kp * 8, 256) + rup((ntail * 4 + 64) * 8, 256);
  return std::max(b, polar_workspace_bytes(v, k)) + 4096;
}

int srm_gemm_tn(const double* w, int64_t ldw, const void* x, int x_dtype, int64_t ldx, int64_t v, int64_t k,
                int64_t t, double alpha, double* out, int64_t ldo, void* workspace, int64_t ws_bytes,
                void* stream) {
  if (v < 1 || k < 1 || t < 1 || !contract_kp_supported((int)rup(k, 8))) return SRM_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t kp = rup(k, 8), ldxp = rup(t, 32);
  const int64_t es = x_dtype == SRM_F64 ? 8 : 4;
  const int64_t nch = std::max<int64_t>(1, (v + kChunk - 1) / kChunk);
  Carve c{static_cast<char*>(workspace), 0, ws_bytes};
  double* Lp = c.take<double>(v * kp);
  char* Xp = c.take<char>(v * ldxp * es);
  double* part = c.take<double>(nch * kp * ldxp);
  double* red = c.take<double>(kp * ldxp);
  ItemE* items = c.take<ItemE>(nch * ((ldxp + 127) / 128));
  if (!items) return SRM_ERR_CONFIG;
  cudaError_t e = cudaMemsetAsync(Lp, 0, v * kp * 8, st);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(Lp, kp * 8, w, ldw * 8, k * 8, v, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(Xp, 0, v * ldxp * es, st);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(Xp, ldxp * es, x, ldx * es, t * es, v, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = split_v(Lp, kp, Xp, x_dtype, ldxp, ldxp, v, alpha, part, red, items, st);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(out, ldo * 8, red, ldxp * 8, t * 8, k, cudaMemcpyDeviceToDevice, st);
  return ret(e);
}

int srm_gemm_nt(const void* x, int x_dtype, int64_t ldx, const double* s, int64_t lds, int64_t v, int64_t t,
                int64_t k, double alpha, double* out, int64_t ldo, void* workspace, int64_t ws_bytes,
                void* stream) {
  if (v < 1 || k < 1 || t < 1 || !contract_kp_supported((int)rup(k, 8))) return SRM_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t kp = rup(k, 8), ldxp = rup(t, 32);
  const int64_t es = x_dtype == SRM_F64 ? 8 : 4;
  Carve c{static_cast<char*>(workspace), 0, ws_bytes};
  char* Xp = c.take<char>(v * ldxp * es);
  double* Sp = c.take<double>(kp * ldxp);
  double* Op = c.take<double>(v * kp);
  ItemA* items = c.take<ItemA>((v + 127) / 128);
  if (!items) return SRM_ERR_CONFIG;
  std::vector<ItemA> host;
  for (int64_t r = 0; r < v; r += 128) {
    ItemA it;
    it.x_off = r * ldxp;
    it.o_off = r * kp;
    it.rows = (int32_t)std::min<int64_t>(128, v - r);
    it.pad = 0;
    host.push_back(it);
  }
  const char* where = "gemm_nt: stage X";
  cudaError_t e = cudaMemsetAsync(Xp, 0, v * ldxp * es, st);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(Xp, ldxp * es, x, ldx * es, t * es, v, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) { where = "gemm_nt: stage S"; e = cudaMemsetAsync(Sp, 0, kp * ldxp * 8, st); }
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(Sp, ldxp * 8, s, lds * 8, t * 8, k, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) { where = "gemm_nt: items"; e = cudaMemcpyAsync(items, host.data(), host.size() * sizeof(ItemA), cudaMemcpyHostToDevice, st); }
  if (e == cudaSuccess) {
    where = "gemm_nt: contract_a";
    e = launch_contract_a((int)kp, x_dtype, Xp, ldxp, Sp, ldxp, ldxp, Op, kp, alpha, items, (int)host.size(), st);
  }
  if (e == cudaSuccess) { where = "gemm_nt: copy out"; e = cudaMemcpy2DAsync(out, ldo * 8, Op, kp * 8, k * 8, v, cudaMemcpyDeviceToDevice, st); }
  return ret(e, where);
}

int srm_project(const double* w, int64_t ldw, const void* x, int x_dtype, int64_t ldx, const double* mu, int64_t v,
                int64_t k, int64_t t, double* out, int64_t ldo, void* workspace, int64_t ws_bytes, void* stream) {
  if (v < 1 || k < 1 || t < 1 || !contract_kp_supported((int)rup(k, 8))) return SRM_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t kp = rup(k, 8), ldxp = rup(t, 32);
  const int64_t nch = std::max<int64_t>(1, (v + kChunk - 1) / kChunk);
  Carve c{static_cast<char*>(workspace), 0, ws_bytes};
  double* Lp = c.take<double>(v * kp);
  double* Xp = c.take<double>(v * ldxp);
  double* part = c.take<double>(nch * kp * ldxp);
  double* red = c.take<double>(kp * ldxp);
  ItemE* items = c.take<ItemE>(nch * ((ldxp + 127) / 128));
  if (!items) return SRM_ERR_CONFIG;
  cudaError_t e = cudaMemsetAsync(Lp, 0, v * kp * 8, st);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(Lp, kp * 8, w, ldw * 8, k * 8, v, cudaMemcpyDeviceToDevice, st);
  // the centering (srm.py:333 x - mu) fused into the fp64 staging copy of X
  if (e == cudaSuccess) e = launch_center_stage(x, x_dtype, ldx, mu, v, t, Xp, ldxp, st);
  if (e == cudaSuccess) e = split_v(Lp, kp, Xp, SRM_F64, ldxp, ldxp, v, 1.0, part, red, items, st);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(out, ldo * 8, red, ldxp * 8, t * 8, k, cudaMemcpyDeviceToDevice, st);
  return ret(e, "project");
}

int srm_unproject(const double* w, int64_t ldw, const double* z, int64_t ldz, const double* mu, int64_t v, int64_t k,
                  int64_t t, double* out, int64_t ldo, void* stream) {
  if (v < 1 || k < 1 || t < 1) return SRM_ERR_SHAPE;
  if (!gemm_nn_bias_supported((int)k)) return SRM_ERR_UNSUPPORTED;
  return ret(launch_gemm_nn_bias(w, ldw, z, ldz, mu, out, ldo, v, (int)k, t, static_cast<cudaStream_t>(stream)),
             "unproject");
}

int srm_tail_step(const double* reduced, int64_t ldr, const double* sigma, int64_t ldsig, int64_t k, int64_t t,
                  double rho0, double* s_out, int64_t lds_out, double* var_out, double* sigma_out,
                  double* trace_out, int32_t* status4, void* workspace, int64_t ws_bytes, void* stream) {
  if (k < 1 || t < 1) return SRM_ERR_SHAPE;
  if (k > max_supported_k()) return SRM_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t kp = rup(k, 8), ldx = rup(t, 32);
  const int ntail = (int)(ldx / 32);
  Carve c{static_cast<char*>(workspace), 0, ws_bytes};
  DevPlan d{};
  d.T = t;
  d.K = k;
  d.ldx = ldx;
  d.kp = kp;
  d.ldo = ldx + kp;
  d.ntile_tail = ntail;
  d.apply_cols = apply_cols_for(kp);
  d.ntile_apply = (int)((ldx + d.apply_cols - 1) / d.apply_cols);
  d.red_stride = kp * ldx + kRedScalars;
  d.hist_stride = 8;
  d.n_hist = 1;
  d.red = c.take<double>(d.red_stride);
  d.S = c.take<double>(kp * ldx);
  d.sigma = c.take<double>(kp * kp);
  d.sinv = c.take<double>(kp * kp);
  d.var = c.take<double>(kp * kp);
  d.cmat = c.take<double>(kp * kp);
  d.sspart = c.take<double>(ntail * kp * kp);
  d.tailpart = c.take<double>(ntail * 4);
  d.tailscr = c.take<double>(kTailScalars);
  d.hist = c.take<double>(8);
  d.iter = c.take<int32_t>(4);
  d.status = status4;
  if (!d.iter) return SRM_ERR_CONFIG;
  cudaError_t e = cudaMemsetAsync(workspace, 0, c.used, st);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(d.red, ldx * 8, reduced, ldr * 8, t * 8, k, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d.red + kp * ldx + RD_RHO0, &rho0, 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(d.sigma, kp * 8, sigma, ldsig * 8, k * 8, k, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = launch_tail(d, st);
  if (e == cudaSuccess && s_out) e = cudaMemcpy2DAsync(s_out, lds_out * 8, d.S, ldx * 8, t * 8, k, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && var_out) e = cudaMemcpy2DAsync(var_out, k * 8, d.var, kp * 8, k * 8, k, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && sigma_out) e = cudaMemcpy2DAsync(sigma_out, k * 8, d.sigma, kp * 8, k * 8, k, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && trace_out) e = cudaMemcpyAsync(trace_out, d.tailscr + TS_TRACE, 8, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // rho0 staged from the caller's stack
  return ret(e);
}

int srm_trace_ata(const double* a, int64_t lda, int64_t rows, int64_t cols, double* out, int32_t* status4,
                  void* workspace, int64_t ws_bytes, void* stream) {
  if (rows < 1 || cols < 1 || lda < cols) return SRM_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = rows * cols;
  const int nct = (int)std::min<int64_t>(1024, (n + 4095) / 4096);
  const int64_t per = (n + nct - 1) / nct;
  if (ws_bytes < nct * 8) return SRM_ERR_CONFIG;
  double* part = static_cast<double*>(workspace);
  k_sumsq_part<<<nct, kSqThreads, 0, st>>>(a, lda, rows, cols, per, part, status4);
  k_sum_final<<<1, kSqThreads, 0, st>>>(part, nct, out);
  return ret(cudaGetLastError(), "trace_ata");
}

int srm_dot(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t rows, int64_t cols, double* out,
            void* workspace, int64_t ws_bytes, void* stream) {
  if (rows < 1 || cols < 1 || lda < cols || ldb < cols) return SRM_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = rows * cols;
  const int nct = (int)std::min<int64_t>(1024, (n + 4095) / 4096);
  const int64_t per = (n + nct - 1) / nct;
  if (ws_bytes < nct * 8) return SRM_ERR_CONFIG;
  double* part = static_cast<double*>(workspace);
  k_dot_part<<<nct, kSqThreads, 0, st>>>(a, lda, b, ldb, rows, cols, per, part);
  k_sum_final<<<1, kSqThreads, 0, st>>>(part, nct, out);
  return ret(cudaGetLastError(), "dot");
}

int srm_sigma_update(const double* var, int64_t ldv, const double* ss, int64_t ldss, int64_t k, int64_t t,
                     double* out, int64_t ldo, double* trace_out, void* stream) {
  if (k < 1 || t < 1) return SRM_ERR_SHAPE;
  k_sigma_update<<<1, kSqThreads, 0, static_cast<cudaStream_t>(stream)>>>(var, ldv, ss, ldss, (int)k, 1.0 / (double)t,
                                                                         out, ldo, trace_out);
  return ret(cudaGetLastError(), "sigma_update");
}

int srm_add_diag(const double* a, int64_t lda, int64_t n, double c, double* out, int64_t ldo, void* stream) {
  if (n < 1 || lda < n || ldo < n) return SRM_ERR_SHAPE;
  const int64_t tot = n * n;
  k_add_diag<<<(unsigned)((tot + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(a, lda, n, c, out, ldo);
  return ret(cudaGetLastError(), "add_diag");
}

int srm_spd_inverse(double* a, int64_t n, int32_t* status4, void* stream) {
  if (n < 1 || n > max_supported_k()) return n < 1 ? SRM_ERR_SHAPE : SRM_ERR_UNSUPPORTED;
  return ret(launch_spd_inverse(a, (int)n, status4, static_cast<cudaStream_t>(stream)));
}

int srm_polar(const double* a, int64_t lda, int64_t v, int64_t k, double* w, int64_t ldw, int32_t* status4,
              void* workspace, int64_t ws_bytes, void* stream) {
  if (v < k) return SRM_ERR_SHAPE;
  if (k < 1) return SRM_ERR_SHAPE;
  if (k > max_supported_k() || !qr_polar_supported((int)k)) return SRM_ERR_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t kp = rup(k, 8);
  const int64_t nch = std::max<int64_t>(1, (v + kChunk - 1) / kChunk);
  const TsqrSchedule sch = tsqr_schedule({v}, (int)k, kPolarCtas);
  Carve c{static_cast<char*>(workspace), 0, ws_bytes};
  double* Ap = c.take<double>(v * kp);
  double* Wt = c.take<double>(v * kp);
  double* rb0 = c.take<double>(sch.buf_doubles);
  double* rb1 = c.take<double>(sch.buf_doubles);
  double* part = c.take<double>(nch * kp * kp);
  double* G = c.take<double>(kp * kp);
  double* M = c.take<double>(kp * kp);
  double* M2 = c.take<double>(kp * kp);
  double* Vg = c.take<double>(kp * kp);
  QrJob* qj = c.take<QrJob>((int64_t)sch.levels.size());
  SvdJob* sj = c.take<SvdJob>(1);
  ItemE* items = c.take<ItemE>(nch);
  if (!items) return SRM_ERR_CONFIG;
  // (1) R of A = Q R (Householder TSQR), (2) SVD of R (one-sided Jacobi) ->
  // M = V diag(1/sigma) V^T and the rank test of kernels.py:202-206, (3) W = A M
  // (the polar factor up to eps cond(A)), (4) one exact polar step of W itself,
  // W <- W (W^T W)^{-1/2}: W^T W is within eps cond(A) of I, so this restores
  // orthonormality to fp64 roundoff (W = U V^T of gesdd is orthonormal to eps)
  std::vector<const double*> rfin;
  const std::vector<std::vector<QrJob>> jobs = tsqr_jobs(sch, {Ap}, {kp}, (int)k, rb0, rb1, &rfin);
  std::vector<QrJob> flat;
  for (const auto& l : jobs) flat.push_back(l[0]);
  const char* where = "polar: stage A";
  cudaError_t e = cudaMemsetAsync(Ap, 0, v * kp * 8, st);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(Ap, kp * 8, a, lda * 8, k * 8, v, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(qj, flat.data(), flat.size() * sizeof(QrJob), cudaMemcpyHostToDevice, st);
  for (size_t L = 0; L < jobs.size() && e == cudaSuccess; ++L) {
    where = "polar: tsqr";
    e = launch_tsqr(qj + L, 1, tsqr_max_ctas(sch.levels[L]), (int)k, st);
  }
  SvdJob sv{rfin[0], M, kp, (int32_t)kp, 0, svd_needs_global_v((int)k) ? Vg : nullptr};
  if (e == cudaSuccess) { where = "polar: svd"; e = cudaMemcpyAsync(sj, &sv, sizeof(SvdJob), cudaMemcpyHostToDevice, st); }
  if (e == cudaSuccess) e = launch_svd_polar(sj, 1, (int)k, status4, nullptr, st);
  if (e == cudaSuccess) { where = "polar: A M"; e = cudaMemsetAsync(Wt, 0, v * kp * 8, st); }
  if (e == cudaSuccess) e = launch_apply_right(Ap, kp, v, (int)k, M, kp, Wt, kp, st);
  // (4) W <- W (3 I - W^T W) / 2 twice: W^T W is within eps cond(A) of I, and
  // each Newton-Schulz step squares that distance (cond 1e11: 2e-5 -> 6e-10 -> 1e-18)
  for (int step = 0; step < 2 && e == cudaSuccess; ++step) {
    double* src = step == 0 ? Wt : Ap;  // Ap (A) is no longer needed after W = A M
    double* dst = step == 0 ? Ap : w;
    const int64_t ldd = step == 0 ? kp : ldw;
    where = "polar: W^T W";
    e = split_v(src, kp, src, SRM_F64, kp, kp, v, 1.0, part, G, items, st);
    if (e == cudaSuccess) { where = "polar: refine"; e = launch_ns_step_matrix(G, kp, (int)k, M2, kp, st); }
    if (e == cudaSuccess && step == 0) e = cudaMemsetAsync(Ap, 0, v * kp * 8, st);
    if (e == cudaSuccess) e = launch_apply_right(src, kp, v, (int)k, M2, kp, dst, ldd, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the job tables were staged from the host stack
  return ret(e, where);
}

}  // extern "C"
