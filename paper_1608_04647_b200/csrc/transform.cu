// The fitted model's transforms (srm.py:330-338), batched over the columns of
// a block of volumes:
//   project:     Z = W_i^T (X - mu_i 1^T)          (K x T')
//   map_between: Y = W_j Z + mu_j 1^T               (V_j x T')
// The centering is fused into the staging pass that widens X to fp64 (the
// reference subtracts in fp64 before the product, so project(mu_i) == 0
// exactly), the V-contraction is the fit's split-V DMMA kernel, and the
// K-contraction with the mean added back is one DMMA GEMM with a bias epilogue.
#include "common.cuh"
#include "kernels.h"

namespace srm {

namespace {

template <typename TX>
__global__ void k_center_stage(const TX* __restrict__ x, int64_t ldx, const double* __restrict__ mu, int64_t v,
                               int64_t t, double* __restrict__ xp, int64_t ldp) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= v * ldp) return;
  const int64_t r = e / ldp, c = e - r * ldp;
  xp[e] = c < t ? static_cast<double>(x[r * ldx + c]) - (mu ? mu[r] : 0.0) : 0.0;
}

// out[r][n] = sum_k A[r][k] B[k][n] + bias[r]: 64 x 64 tiles, 8 warps of
// 16 rows x 32 columns on mma.sync.m8n8k4.f64; K <= kMaxKB in shared memory
constexpr int kMaxKB = 128;
constexpr int kGT = 64;
constexpr int kGAld = kMaxKB + 4;  // == 4 mod 16 doubles: conflict-free fragment loads
constexpr int kGBld = kGT + 4;

__global__ void __launch_bounds__(256) k_gemm_nn_bias(const double* __restrict__ A, int64_t lda,
                                                      const double* __restrict__ B, int64_t ldb,
                                                      const double* __restrict__ bias, double* __restrict__ out,
                                                      int64_t ldo, int64_t V, int K, int64_t N) {
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                 // [64][kGAld]
  double* Bs = gsm + kGT * kGAld;   // [kp][kGBld]
  const int64_t r0 = (int64_t)blockIdx.x * kGT, n0 = (int64_t)blockIdx.y * kGT;
  const int kp = (K + 3) & ~3;
  for (int e = threadIdx.x; e < kGT * kp; e += blockDim.x) {
    const int r = e / kp, k = e - r * kp;
    As[r * kGAld + k] = (r0 + r < V && k < K) ? A[(r0 + r) * lda + k] : 0.0;
  }
  for (int e = threadIdx.x; e < kp * kGT; e += blockDim.x) {
    const int k = e / kGT, n = e - k * kGT;
    Bs[k * kGBld + n] = (k < K && n0 + n < N) ? B[(int64_t)k * ldb + n0 + n] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp & 3) * 16, wc = (warp >> 2) * 32;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < kp; k0 += 4) {
    double a[2], b[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) a[i] = As[(wr + i * 8 + (lane >> 2)) * kGAld + k0 + (lane & 3)];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = Bs[(k0 + (lane & 3)) * kGBld + wc + j * 8 + (lane >> 2)];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t r = r0 + wr + i * 8 + (lane >> 2);
    if (r >= V) continue;
    const double bb = bias ? bias[r] : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = n0 + wc + j * 8 + 2 * (lane & 3);
      if (c < N) out[r * ldo + c] = acc[i][j][0] + bb;
      if (c + 1 < N) out[r * ldo + c + 1] = acc[i][j][1] + bb;
    }
  }
}

}  // namespace

cudaError_t launch_center_stage(const void* x, int x_dtype, int64_t ldx, const double* mu, int64_t v, int64_t t,
                                double* xp, int64_t ldp, cudaStream_t st) {
  const int64_t n = v * ldp;
  if (n == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (x_dtype == 0)
    k_center_stage<double><<<grid, 256, 0, st>>>(static_cast<const double*>(x), ldx, mu, v, t, xp, ldp);
  else
    k_center_stage<float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), ldx, mu, v, t, xp, ldp);
  return cudaGetLastError();
}

bool gemm_nn_bias_supported(int K) { return K >= 1 && K <= kMaxKB; }

cudaError_t launch_gemm_nn_bias(const double* A, int64_t lda, const double* B, int64_t ldb, const double* bias,
                                double* out, int64_t ldo, int64_t V, int K, int64_t N, cudaStream_t st) {
  if (!gemm_nn_bias_supported(K)) return cudaErrorInvalidValue;
  const size_t bytes = (size_t)(kGT * kGAld + ((K + 3) & ~3) * kGBld) * sizeof(double);
  static size_t configured = 0;
  if (bytes > 48 * 1024 && bytes > configured) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_nn_bias, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured = bytes;
  }
  if (V == 0 || N == 0) return cudaSuccess;
  const dim3 grid((unsigned)((V + kGT - 1) / kGT), (unsigned)((N + kGT - 1) / kGT));
  k_gemm_nn_bias<<<grid, 256, bytes, st>>>(A, lda, B, ldb, bias, out, ldo, V, K, N);
  return cudaGetLastError();
}

}  // namespace srm
