// Shared device helpers for the SRM EM kernels (sm_100a).
//
// Everything here is plain CUDA C++ / inline PTX for Blackwell; there is no
// portability layer.  fp64 contractions use the FP64 tensor path
// (mma.sync m8n8k4 -> SASS DMMA.8x8x4), which measured 37.1 TFLOP/s on the
// pool's B200 against 33.8 for DFMA (tools/fp64_peak.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/srm_b200.h"

namespace srm {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// device status word: {code, arg (subject / pivot), iteration, warning bits}
// first error wins (atomicCAS on code); later kernels may early-exit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void raise_status(int32_t* status, int code, int arg, int iter) {
  if (atomicCAS(&status[0], 0, code) == 0) {
    status[1] = arg;
    status[2] = iter;
  }
}

// warning bits in status[3] (SRM_WARN_*): sticky, never abort the stream.
// The Gram-route polar transform (A^T A)^{-1/2} cannot resolve
// sigma_min / sigma_max below ~1e-8 and loses ~eps cond(A)^2; when a subject's
// A^T A is that ill-conditioned it sets SRM_WARN_POLAR_CONDITION instead of
// deciding the rank test, and the host re-runs the fit on the exact route
// (TSQR + SVD of A, qr_polar.cu), which raises RankError as kernels.py:202-206.
__device__ __forceinline__ void raise_warning(int32_t* status, int bits) { atomicOr(&status[3], bits); }
// largest c / lambda_min (c >= lambda_max) the Gram route accepts: the
// transform's error ~eps_G c / lambda_min stays below ~1e-9 for the ~1e-14
// relative error eps_G of the int8-sliced Gram
constexpr double kGramCondLimit = 1e5;

// ---------------------------------------------------------------------------
// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col)
//   A fragment: lane holds A[lane/4][lane%4]
//   B fragment: lane holds B[lane%4][lane/4]
//   C fragment: lane holds C[lane/4][2*(lane%4) + {0,1}]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers; zero-fill when the source is out of range.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const int src_size = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src_size));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------
// small reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum (fixed tree); all threads get the result.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  v = warp_sum(v);
  const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (l < NT / kWarp) ? scratch[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) scratch[0] = t;
  }
  __syncthreads();
  t = scratch[0];
  __syncthreads();
  return t;
}

// L2 load of data another CTA wrote before a fence + atomic handshake: a weak
// ld.global.cg (L1 bypassed), so independent loads stay in flight together
__device__ __forceinline__ double ld_cg(const double* ptr) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(ptr));
  return v;
}

template <typename T>
__device__ __forceinline__ double to_f64(T x) { return static_cast<double>(x); }

}  // namespace srm
