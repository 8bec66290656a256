// Polar transform M_i = (A_i^T A_i)^{-1/2} by the coupled Newton-Schulz
// iteration on the FP64 tensor cores (one CTA per subject, K <= 80).
//
// kernels.py:190-212 forms the polar factor W = U V^T from an SVD of A.  For
// full-rank A it equals A (A^T A)^{-1/2}; with C = A^T A scaled by c >= lambda_max
// (Gershgorin bound), the iteration
//     Y_0 = C / c,  Z_0 = I,  T_k = (3 I - Z_k Y_k) / 2,
//     Y_{k+1} = T_k Y_k,  Z_{k+1} = T_k Z_k
// converges quadratically to Y -> (C/c)^{1/2}, Z -> (C/c)^{-1/2} (all iterates
// are polynomials in C, so they commute and stay symmetric).  Each step is three
// K x K products done with mma.sync.m8n8k4.f64 from shared memory, upper tiles
// only (the products are symmetric) -- a
// tensor-core replacement for the latency-bound Jacobi rotations.  A direction
// with lambda ~ 0 converges slowly or not at all, and any lambda_min below
// c / kGramCondLimit is beyond what the Gram route resolves: both raise
// SRM_WARN_POLAR_CONDITION, and the fit is redone on the exact route
// (qr_polar.cu), which applies the rank test of kernels.py:202-206.
#include "common.cuh"
#include "plan.h"

namespace srm {

namespace {

constexpr int kNsThreads = 512;

// The M-step's cross term <W^T Xhat, S> (srm.py:151) from the polar itself:
// with P = M^T B and B S^T = 2 C (C = A^T A as gram_from_b stores it, before
// symmetrisation), <P, S> = tr(M^T B S^T) = 2 sum_{c,f} M[c][f] C[c][f] -- a
// K x K dot product here instead of a reduction over apply_m's K x T tiles, so
// rho_i^2 (finalize_rho) no longer waits for apply_m (DevPlan::polar_cross).
// `cr` is this thread's part of sum M C; every thread of the block calls this.
__device__ __forceinline__ void polar_cross_out(const DevPlan& p, int i, double cr, double* red) {
  cr = block_sum<kNsThreads>(cr, red);
  for (int t = threadIdx.x; t < p.ntile_apply; t += blockDim.x)
    p.crossp[(int64_t)i * p.ntile_apply + t] = t == 0 ? 2.0 * cr : 0.0;
}

__host__ __device__ constexpr int ns_ld(int kp) { return kp + ((4 - kp) % 16 + 16) % 16; }

// D = A * B for symmetric products (A, B commuting polynomials in C): only
// the NT (NT + 1) / 2 upper 8 x 8 tiles are computed, split evenly over the
// warps (consecutive tiles, so a warp's tiles share row strips), with every
// tile's k-chain interleaved; `epi(row, col, v0, v1, diag)` consumes
// D[row][col..col+1] and stores the mirrored entries itself.
template <int KP>
struct SymTiles {
  static constexpr int NT = KP / 8;
  static constexpr int N = NT * (NT + 1) / 2;
  static constexpr int W = kNsThreads / 32;
  static constexpr int PER = (N + W - 1) / W;
};

template <int KP, typename Epi>
__device__ __forceinline__ void mm_sym(const double* __restrict__ A, const double* __restrict__ B, Epi epi) {
  constexpr int LD = ns_ld(KP);
  using TL = SymTiles<KP>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tm[TL::PER], tn[TL::PER];
  bool on[TL::PER];
#pragma unroll
  for (int q = 0; q < TL::PER; ++q) {
    // upper tile index -> (m, n), m <= n, row-major over the upper triangle
    int idx = warp * TL::PER + q, m = 0;
    on[q] = idx < TL::N;
    if (!on[q]) idx = 0;
    while (idx >= TL::NT - m) {
      idx -= TL::NT - m;
      ++m;
    }
    tm[q] = m;
    tn[q] = m + idx;
  }
  double acc[TL::PER][2];
#pragma unroll
  for (int q = 0; q < TL::PER; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll 2
  for (int k0 = 0; k0 < KP; k0 += 4) {
#pragma unroll
    for (int q = 0; q < TL::PER; ++q) {
      if (on[q]) {
        const double a = A[(tm[q] * 8 + (lane >> 2)) * LD + k0 + (lane & 3)];
        const double b = B[(k0 + (lane & 3)) * LD + tn[q] * 8 + (lane >> 2)];
        dmma(acc[q][0], acc[q][1], a, b);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < TL::PER; ++q)
    if (on[q]) epi(tm[q] * 8 + (lane >> 2), tn[q] * 8 + 2 * (lane & 3), acc[q][0], acc[q][1], tm[q] == tn[q]);
}

template <int KP>
__global__ void __launch_bounds__(kNsThreads) k_ns_polar(DevPlan p, int init) {
  constexpr int LD = ns_ld(KP);
  constexpr int MAT = KP * LD;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32];
  __shared__ double s_scale;
  const int i = p.sub0 + blockIdx.x;
  const int n = (int)p.K;
  const int tid = threadIdx.x;
  double* buf[4] = {sm, sm + MAT, sm + 2 * MAT, sm + 3 * MAT};
  const double* Cg = p.bred + (int64_t)i * p.kp * p.ldo + p.ldx;  // A^T A block, row stride ldo

  // C staged in buf[2] (eight loads in flight per thread), then Y0 = sym(C) / c
  // (c: Gershgorin bound on lambda_max), Z0 = I; pads are zero
  double* Cs = buf[2];
  for (int e0 = 0; e0 < KP * KP; e0 += 8 * kNsThreads) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * kNsThreads;
      const int a = e / KP, b = e - a * KP;
      v[u] = (e < KP * KP && a < n && b < n) ? Cg[(int64_t)a * p.ldo + b] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + tid + u * kNsThreads;
      if (e < KP * KP) Cs[(e / KP) * LD + e % KP] = v[u];
    }
  }
  __syncthreads();
  double rowmax = 0.0;
  for (int a = tid; a < KP; a += blockDim.x) {
    double rs = 0.0;
    for (int b = 0; b < n && a < n; ++b) rs += fabs(0.5 * (Cs[a * LD + b] + Cs[b * LD + a]));
    rowmax = fmax(rowmax, rs);
  }
  rowmax = warp_max(rowmax);
  if ((tid & 31) == 0) red[tid >> 5] = rowmax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < kNsThreads / 32; ++w) m = fmax(m, red[w]);
    s_scale = m;
  }
  __syncthreads();
  const double c = s_scale;
  const bool degenerate = !(c > 0.0) || !isfinite(c);
  const double inv_c = degenerate ? 0.0 : 1.0 / c;
  for (int e = tid; e < KP * LD; e += blockDim.x) {
    const int a = e / LD, b = e - a * LD;
    double y = 0.0;
    if (a < n && b < n) y = 0.5 * (Cs[a * LD + b] + Cs[b * LD + a]) * inv_c;
    buf[0][e] = y;
    buf[1][e] = (a == b && a < n) ? 1.0 : 0.0;
  }
  __syncthreads();

  int y = 0, z = 1;  // buffer indices of Y and Z
  bool converged = false;
  int extra = -1;
  double prev_err = 1e300;
  const int max_iter = 90;
  int it = 0;
  for (; it < max_iter && !degenerate; ++it) {
    // free buffers: the two not holding Y or Z
    int f0 = -1, f1 = -1;
    for (int q = 0; q < 4; ++q)
      if (q != y && q != z) (f0 < 0 ? f0 : f1) = q;
    double* Tm = buf[f0];
    double* Yn = buf[f1];
    // P = Z Y -> T = (3I - P)/2 in place, and |I - P|_F^2 (P is symmetric:
    // off-diagonal tiles count twice)
    double err = 0.0;
    mm_sym<KP>(buf[z], buf[y], [&](int r, int col, double v0, double v1, bool dg) {
      const double d0 = (r == col ? 1.0 : 0.0) - v0, d1 = (r == col + 1 ? 1.0 : 0.0) - v1;
      const double wgt = dg ? 1.0 : 2.0;
      if (r < n && col < n) err += wgt * d0 * d0;
      if (r < n && col + 1 < n) err += wgt * d1 * d1;
      const double t0 = 0.5 * (r == col ? 3.0 - v0 : -v0), t1 = 0.5 * (r == col + 1 ? 3.0 - v1 : -v1);
      Tm[r * LD + col] = t0;
      Tm[r * LD + col + 1] = t1;
      if (!dg) {
        Tm[col * LD + r] = t0;
        Tm[(col + 1) * LD + r] = t1;
      }
    });
    err = block_sum<kNsThreads>(err, red);  // includes a barrier: T is complete
    if (extra == 0) {
      converged = true;
      break;
    }
    if (!(err == err)) break;  // NaN
    // |I - P|_F <= 1e-10 (quadratic convergence: one more step reaches the
    // roundoff floor), or the floor is already hit (|I - P| no longer shrinking
    // while below 1e-9): one more step, then stop
    if (extra < 0 && (err <= 1e-20 || (err < 1e-18 && err > 0.25 * prev_err))) extra = 1;
    prev_err = err;
    // Y_new = T Y  (-> Yn),  Z_new = T Z (-> old Y buffer once Y is consumed)
    mm_sym<KP>(Tm, buf[y], [&](int r, int col, double v0, double v1, bool dg) {
      Yn[r * LD + col] = v0;
      Yn[r * LD + col + 1] = v1;
      if (!dg) {
        Yn[col * LD + r] = v0;
        Yn[(col + 1) * LD + r] = v1;
      }
    });
    __syncthreads();
    double* Zn = buf[y];
    mm_sym<KP>(Tm, buf[z], [&](int r, int col, double v0, double v1, bool dg) {
      Zn[r * LD + col] = v0;
      Zn[r * LD + col + 1] = v1;
      if (!dg) {
        Zn[col * LD + r] = v0;
        Zn[(col + 1) * LD + r] = v1;
      }
    });
    __syncthreads();
    z = y;   // Z now lives in the old Y buffer
    y = f1;  // Y in Yn
    if (extra > 0 && --extra == 0) {
      ++it;
      converged = true;  // the step after the trigger: no check product needed
      break;
    }
  }
  // M = sym(Z) / sqrt(c); |Z|_F^2 = sum_j c / lambda_j >= c / lambda_min
  const int kp = (int)p.kp;
  double* Mg = p.mmat + (int64_t)i * kp * kp;
  const double* Z = buf[z];
  const double s = degenerate ? 0.0 : 1.0 / sqrt(c);
  double zz = 0.0, cr = 0.0;
  const bool want_cross = p.polar_cross && !init;
  for (int e = tid; e < kp * kp; e += blockDim.x) {
    const int a = e / kp, b = e - a * kp;
    const double v = (a < n && b < n) ? 0.5 * (Z[a * LD + b] + Z[b * LD + a]) : 0.0;
    zz = fma(v, v, zz);
    Mg[e] = v * s;
    if (want_cross && a < n && b < n) cr = fma(v * s, Cg[(int64_t)a * p.ldo + b], cr);
  }
  zz = block_sum<kNsThreads>(zz, red);
  if (want_cross) polar_cross_out(p, i, cr, red);
  if (tid == 0) {
    p.scal[(int64_t)i * 8 + 0] = (double)it;
    if (degenerate || !converged || !(zz <= kGramCondLimit)) raise_warning(p.status, SRM_WARN_POLAR_CONDITION);
  }
}

template <int KP>
cudaError_t run_ns(const DevPlan& p, int init, cudaStream_t s) {
  constexpr int bytes = 4 * KP * ns_ld(KP) * (int)sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_ns_polar<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k_ns_polar<KP><<<p.nsub, kNsThreads, bytes, s>>>(p, init);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// The same fp64 coupled iteration for 80 < kp <= 128, where four K x K fp64
// matrices no longer fit in shared memory: Y, Z, T and Y' live in a per-subject
// global scratch (4 kp^2 doubles, L2-resident) and every product streams
// 32-wide k-slabs of its operands through shared memory into DMMA fragments.
// fp64 throughout, so the transform is as accurate as the kp <= 80 kernel's
// (an fp32 iteration carried ~4e-7 into S per iteration).
// ---------------------------------------------------------------------------
// k-slab of the staged operands: the whole matrix while two fit in shared
// memory (kp <= 112: one round of loads, all in flight), else 64 wide
template <int KP>
struct NsgSlab {
  static constexpr int W = KP <= 112 ? KP : 64;
  static constexpr int LDA = ns_ld(W);  // == 4 mod 16 doubles: conflict-free fragments
};

template <int KP, typename Epi>
__device__ __forceinline__ void gmm_sym(const double* A, const double* B, double* As, double* Bs, Epi epi) {
  constexpr int LDB = ns_ld(KP);
  constexpr int kSlab = NsgSlab<KP>::W;
  constexpr int kSlabLd = NsgSlab<KP>::LDA;
  using TL = SymTiles<KP>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tm[TL::PER], tn[TL::PER];
  bool on[TL::PER];
#pragma unroll
  for (int q = 0; q < TL::PER; ++q) {
    int idx = warp * TL::PER + q, m = 0;
    on[q] = idx < TL::N;
    if (!on[q]) idx = 0;
    while (idx >= TL::NT - m) {
      idx -= TL::NT - m;
      ++m;
    }
    tm[q] = m;
    tn[q] = m + idx;
  }
  double acc[TL::PER][2];
#pragma unroll
  for (int q = 0; q < TL::PER; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int k0 = 0; k0 < KP; k0 += kSlab) {
    const int kw = min(kSlab, KP - k0);
    // 16-byte cp.async (LDGSTS) copies from L2, ~20 per thread in flight at
    // kp = 104 (scalar loads held one or two: the staging was 60% of the kernel)
    constexpr int ca = kSlab / 2, cb = KP / 2;
    for (int e = threadIdx.x; e < KP * ca; e += kNsThreads) {
      const int r = e / ca, kk = 2 * (e - r * ca);
      const bool ok = kk < kw;
      cp_async16(As + r * kSlabLd + kk, A + r * KP + k0 + (ok ? kk : 0), ok);
    }
    for (int e = threadIdx.x; e < kSlab * cb; e += kNsThreads) {
      const int kk = e / cb, c = 2 * (e - kk * cb);
      const bool ok = kk < kw;
      cp_async16(Bs + kk * LDB + c, B + (ok ? (k0 + kk) * KP + c : 0), ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll 2
    for (int kk = 0; kk < kw; kk += 4) {
#pragma unroll
      for (int q = 0; q < TL::PER; ++q) {
        if (on[q]) {
          const double a = As[(tm[q] * 8 + (lane >> 2)) * kSlabLd + kk + (lane & 3)];
          const double b = Bs[(kk + (lane & 3)) * LDB + tn[q] * 8 + (lane >> 2)];
          dmma(acc[q][0], acc[q][1], a, b);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < TL::PER; ++q)
    if (on[q]) epi(tm[q] * 8 + (lane >> 2), tn[q] * 8 + 2 * (lane & 3), acc[q][0], acc[q][1], tm[q] == tn[q]);
}

template <int KP>
__global__ void __launch_bounds__(kNsThreads) k_ns_polar_g(DevPlan p, int init) {
  constexpr int LDB = ns_ld(KP);
  constexpr int MAT = KP * KP;
  extern __shared__ __align__(16) double gsm[];
  __shared__ double red[32];
  __shared__ double s_scale;
  double* As = gsm;                              // [KP][slab pitch]
  double* Bs = gsm + KP * NsgSlab<KP>::LDA;      // [slab][LDB]
  const int i = p.sub0 + blockIdx.x;
  const int n = (int)p.K;
  const int tid = threadIdx.x;
  double* buf[4];
  for (int q = 0; q < 4; ++q) buf[q] = p.nsg + ((int64_t)i * 4 + q) * MAT;
  const double* Cg = p.bred + (int64_t)i * p.kp * p.ldo + p.ldx;  // A^T A block, row stride ldo

  double rowmax = 0.0;
  for (int a = tid >> 2; a < KP; a += kNsThreads / 4) {  // four lanes per row, summed in a fixed order
    double rs = 0.0;
    for (int b = (tid & 3); b < n && a < n; b += 4) rs += fabs(0.5 * (Cg[(int64_t)a * p.ldo + b] + Cg[(int64_t)b * p.ldo + a]));
    rs += __shfl_xor_sync(0xffffffffu, rs, 1);
    rs += __shfl_xor_sync(0xffffffffu, rs, 2);
    rowmax = fmax(rowmax, rs);
  }
  rowmax = warp_max(rowmax);
  if ((tid & 31) == 0) red[tid >> 5] = rowmax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < kNsThreads / 32; ++w) m = fmax(m, red[w]);
    s_scale = m;
  }
  __syncthreads();
  const double c = s_scale;
  const bool degenerate = !(c > 0.0) || !isfinite(c);
  const double inv_c = degenerate ? 0.0 : 1.0 / c;
  for (int e = tid; e < MAT; e += kNsThreads) {
    const int a = e / KP, b = e - a * KP;
    buf[0][e] = (a < n && b < n) ? 0.5 * (Cg[(int64_t)a * p.ldo + b] + Cg[(int64_t)b * p.ldo + a]) * inv_c : 0.0;
    buf[1][e] = (a == b && a < n) ? 1.0 : 0.0;
  }
  __syncthreads();

  int y = 0, z = 1;
  bool converged = false;
  int extra = -1;
  double prev_err = 1e300;
  int it = 0;
  for (; it < 90 && !degenerate; ++it) {
    int f0 = -1, f1 = -1;
    for (int q = 0; q < 4; ++q)
      if (q != y && q != z) (f0 < 0 ? f0 : f1) = q;
    double* Tm = buf[f0];
    double* Yn = buf[f1];
    double err = 0.0;
    gmm_sym<KP>(buf[z], buf[y], As, Bs, [&](int r, int col, double v0, double v1, bool dg) {
      const double d0 = (r == col ? 1.0 : 0.0) - v0, d1 = (r == col + 1 ? 1.0 : 0.0) - v1;
      const double wgt = dg ? 1.0 : 2.0;
      if (r < n && col < n) err += wgt * d0 * d0;
      if (r < n && col + 1 < n) err += wgt * d1 * d1;
      const double t0 = 0.5 * (r == col ? 3.0 - v0 : -v0), t1 = 0.5 * (r == col + 1 ? 3.0 - v1 : -v1);
      Tm[r * KP + col] = t0;
      Tm[r * KP + col + 1] = t1;
      if (!dg) {
        Tm[col * KP + r] = t0;
        Tm[(col + 1) * KP + r] = t1;
      }
    });
    err = block_sum<kNsThreads>(err, red);  // barrier: T is complete
    if (extra == 0) {
      converged = true;
      break;
    }
    if (!(err == err)) break;
    if (extra < 0 && (err <= 1e-20 || (err < 1e-18 && err > 0.25 * prev_err))) extra = 1;
    prev_err = err;
    gmm_sym<KP>(Tm, buf[y], As, Bs, [&](int r, int col, double v0, double v1, bool dg) {
      Yn[r * KP + col] = v0;
      Yn[r * KP + col + 1] = v1;
      if (!dg) {
        Yn[col * KP + r] = v0;
        Yn[(col + 1) * KP + r] = v1;
      }
    });
    __syncthreads();
    double* Zn = buf[y];
    gmm_sym<KP>(Tm, buf[z], As, Bs, [&](int r, int col, double v0, double v1, bool dg) {
      Zn[r * KP + col] = v0;
      Zn[r * KP + col + 1] = v1;
      if (!dg) {
        Zn[col * KP + r] = v0;
        Zn[(col + 1) * KP + r] = v1;
      }
    });
    __syncthreads();
    z = y;
    y = f1;
    if (extra > 0 && --extra == 0) {
      ++it;
      converged = true;
      break;
    }
  }
  const int kp = (int)p.kp;
  double* Mg = p.mmat + (int64_t)i * kp * kp;
  const double* Z = buf[z];
  const double sc = degenerate ? 0.0 : 1.0 / sqrt(c);
  double zz = 0.0, cr = 0.0;
  const bool want_cross = p.polar_cross && !init;
  const double* Cx = p.bred + (int64_t)i * p.kp * p.ldo + p.ldx;
  for (int e = tid; e < kp * kp; e += kNsThreads) {
    const int a = e / kp, b = e - a * kp;
    const double v = (a < n && b < n) ? 0.5 * (Z[a * KP + b] + Z[b * KP + a]) : 0.0;
    zz = fma(v, v, zz);
    Mg[e] = v * sc;
    if (want_cross && a < n && b < n) cr = fma(v * sc, Cx[(int64_t)a * p.ldo + b], cr);
  }
  zz = block_sum<kNsThreads>(zz, red);
  if (want_cross) polar_cross_out(p, i, cr, red);
  if (tid == 0) {
    p.scal[(int64_t)i * 8 + 0] = (double)it;
    if (degenerate || !converged || !(zz <= kGramCondLimit)) raise_warning(p.status, SRM_WARN_POLAR_CONDITION);
  }
}

template <int KP>
cudaError_t run_ns_g(const DevPlan& p, int init, cudaStream_t s) {
  constexpr int bytes = (KP * NsgSlab<KP>::LDA + NsgSlab<KP>::W * ns_ld(KP)) * (int)sizeof(double);
  if (!p.nsg) return cudaErrorInvalidValue;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_ns_polar_g<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k_ns_polar_g<KP><<<p.nsub, kNsThreads, bytes, s>>>(p, init);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// fp32 SIMT variant for the tensor-core (fp32 X-hat) plans with 80 < kp <= 112:
// the same coupled iteration with fp32 matrices (4 x kp x (kp+4) floats fit in
// smem where fp64 does not).  The per-iteration M then carries ~1e-6 relative
// error -- the 3xTF32 passes already do -- and srm_finalize recomputes the
// polar transform exactly (fp64 Jacobi) for the returned W.
// ---------------------------------------------------------------------------
template <int KP>
__device__ __forceinline__ void mm_f32(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
                                       float diag_shift, float scale) {
  // C = scale * (diag_shift * I - A B)  when diag_shift != 0, else C = A B
  constexpr int LD = KP + 4;
  constexpr int R = KP / 16;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[R][R];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) acc[i][j] = 0.f;
  for (int k = 0; k < KP; ++k) {
    float a[R], b[R];
#pragma unroll
    for (int i = 0; i < R; ++i) a[i] = A[(ty + 16 * i) * LD + k];
#pragma unroll
    for (int j = 0; j < R; ++j) b[j] = B[k * LD + tx + 16 * j];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int j = 0; j < R; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int r = ty + 16 * i, c = tx + 16 * j;
      C[r * LD + c] = diag_shift != 0.f ? scale * ((r == c ? diag_shift : 0.f) - acc[i][j]) : acc[i][j];
    }
}

template <int KP>
__global__ void __launch_bounds__(256) k_ns_polar_f32(DevPlan p, int init) {
  constexpr int LD = KP + 4;
  constexpr int MAT = KP * LD;
  extern __shared__ __align__(16) float smf[];
  __shared__ double red[32];
  __shared__ double s_scale;
  const int i = p.sub0 + blockIdx.x;
  const int n = (int)p.K;
  const int tid = threadIdx.x;
  float* buf[4] = {smf, smf + MAT, smf + 2 * MAT, smf + 3 * MAT};
  const double* Cg = p.bred + (int64_t)i * p.kp * p.ldo + p.ldx;
  double rowmax = 0.0;
  for (int a = tid; a < KP; a += blockDim.x) {
    double rs = 0.0;
    for (int b0 = 0; b0 < n && a < n; b0 += 8) {  // eight loads in flight, summed in order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b0 + u;
        v[u] = b < n ? fabs(0.5 * (Cg[(int64_t)a * p.ldo + b] + Cg[(int64_t)b * p.ldo + a])) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (b0 + u < n) rs += v[u];
    }
    rowmax = fmax(rowmax, rs);
  }
  rowmax = warp_max(rowmax);
  if ((tid & 31) == 0) red[tid >> 5] = rowmax;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < 8; ++w) m = fmax(m, red[w]);
    s_scale = m;
  }
  __syncthreads();
  const double c = s_scale;
  const bool degenerate = !(c > 0.0) || !isfinite(c);
  const double inv_c = degenerate ? 0.0 : 1.0 / c;
  for (int e0 = 0; e0 < KP * LD; e0 += 4 * 256) {
    float y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + tid + u * 256;
      const int a = e / LD, b = e - a * LD;
      y[u] = (e < KP * LD && a < n && b < n)
                 ? (float)(0.5 * (Cg[(int64_t)a * p.ldo + b] + Cg[(int64_t)b * p.ldo + a]) * inv_c)
                 : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + tid + u * 256;
      if (e < KP * LD) {
        const int a = e / LD, b = e - a * LD;
        buf[0][e] = y[u];
        buf[1][e] = (a == b && a < n) ? 1.f : 0.f;
      }
    }
  }
  __syncthreads();
  int y = 0, z = 1;
  bool converged = false;
  int extra = -1;
  double prev_err = 1e300;
  int it = 0;
  for (; it < 90 && !degenerate; ++it) {
    int f0 = -1, f1 = -1;
    for (int q = 0; q < 4; ++q)
      if (q != y && q != z) (f0 < 0 ? f0 : f1) = q;
    float* Tm = buf[f0];
    float* Yn = buf[f1];
    mm_f32<KP>(buf[z], buf[y], Tm, 0.f, 1.f);  // P = Z Y
    __syncthreads();
    double err = 0.0;
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int a = e / n, b = e - a * n;
      const double d = (a == b ? 1.0 : 0.0) - (double)Tm[a * LD + b];
      err += d * d;
    }
    err = block_sum<256>(err, red);
    if (extra == 0) {
      converged = true;
      break;
    }
    if (!(err == err)) break;
    if (extra < 0 && (err <= 1e-12 || (err < 1e-8 && err > 0.25 * prev_err))) extra = 1;
    prev_err = err;
    for (int e = tid; e < KP * LD; e += blockDim.x) {  // T = (3I - P)/2 in place
      const int a = e / LD, b = e - a * LD;
      Tm[e] = 0.5f * ((a == b ? 3.f : 0.f) - Tm[e]);
    }
    __syncthreads();
    mm_f32<KP>(Tm, buf[y], Yn, 0.f, 1.f);          // Y' = T Y
    __syncthreads();                                // every thread is done reading Y
    mm_f32<KP>(Tm, buf[z], buf[y], 0.f, 1.f);      // Z' = T Z into the old Y buffer
    __syncthreads();
    z = y;
    y = f1;
    if (extra > 0) --extra;
  }
  const int kp = (int)p.kp;
  double* Mg = p.mmat + (int64_t)i * kp * kp;
  const float* Z = buf[z];
  const double sc = degenerate ? 0.0 : 1.0 / sqrt(c);
  double zz = 0.0;
  for (int e = tid; e < kp * kp; e += blockDim.x) {
    const int a = e / kp, b = e - a * kp;
    const double v = (a < n && b < n) ? 0.5 * ((double)Z[a * LD + b] + (double)Z[b * LD + a]) : 0.0;
    zz = fma(v, v, zz);
    Mg[e] = v * sc;
  }
  zz = block_sum<256>(zz, red);
  if (tid == 0) {
    p.scal[(int64_t)i * 8 + 0] = (double)it;
    if (degenerate || !converged || !(zz <= kGramCondLimit)) raise_warning(p.status, SRM_WARN_POLAR_CONDITION);
  }
}

template <int KP>
cudaError_t run_ns_f32(const DevPlan& p, int init, cudaStream_t s) {
  constexpr int bytes = 4 * KP * (KP + 4) * (int)sizeof(float);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_ns_polar_f32<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k_ns_polar_f32<KP><<<p.nsub, 256, bytes, s>>>(p, init);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Final fp64 polar transform for fp32 X-hat with 80 < kp <= 112, where the
// per-iteration polar ran as the fp32 Newton-Schulz: refine its M (fp32
// accuracy) by the symmetric Newton iteration for the inverse square root
//     E_k = Z_k C Z_k - I,   Z_{k+1} = Z_k - (Z_k E_k + E_k Z_k) / 4,
// which converges quadratically to the SPD solution of Z C Z = I, i.e.
// C^{-1/2} (kernels.py:190-212 via W = A C^{-1/2}); from |E_0| ~ 1e-6 two
// steps reach the fp64 roundoff floor.  One CTA per subject; each K x K
// product stages its two operands in shared memory (2 x K (K + 1) doubles),
// T and E live in the subject's qscr / qmat scratch, Z in mmat (in place).
// A subject whose iteration does not converge keeps scal[i][1] = 0 and is
// recomputed by the Jacobi kernel that follows (RankError semantics there).
// ---------------------------------------------------------------------------
constexpr int kRefThreads = 512;

// D = op(A) op(B) for n x n row-major operands; `sym_a` stages A as (A + A^T) / 2
__device__ __forceinline__ void ref_mm(const double* A, int64_t lda, bool sym_a, const double* B, int64_t ldb,
                                       double* D, int64_t ldd, int n, double* sa, double* sb) {
  const int ld = n + 1;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int a = e / n, b = e - a * n;
    sa[a * ld + b] = sym_a ? 0.5 * (A[(int64_t)a * lda + b] + A[(int64_t)b * lda + a]) : A[(int64_t)a * lda + b];
    sb[a * ld + b] = B[(int64_t)a * ldb + b];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int a = e / n, b = e - a * n;
    double acc = 0.0;
    for (int c = 0; c < n; ++c) acc = fma(sa[a * ld + c], sb[c * ld + b], acc);
    D[(int64_t)a * ldd + b] = acc;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kRefThreads, 1) k_ns_refine(DevPlan p, int warn) {
  extern __shared__ __align__(16) double rsm[];
  __shared__ double red[kRefThreads / 32];
  const int i = p.sub0 + blockIdx.x;
  const int n = (int)p.K, kp = (int)p.kp;
  double* sa = rsm;
  double* sb = rsm + n * (n + 1);
  const double* C = p.bred + (int64_t)i * p.kp * p.ldo + p.ldx;  // A^T A of the last M-step
  double* Z = p.mmat + (int64_t)i * kp * kp;
  double* T = p.qscr + (int64_t)i * kp * kp;
  double* E = p.qmat + (int64_t)i * kp * kp;
  bool ok = false;
  int extra = -1;
  double prev = 1e300;
  int step = 0;
  for (; step < 24; ++step) {
    ref_mm(C, p.ldo, true, Z, kp, T, kp, n, sa, sb);  // T = C Z
    ref_mm(Z, kp, false, T, kp, E, kp, n, sa, sb);    // E = Z C Z (- I below)
    double err = 0.0;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int a = e / n, b = e - a * n;
      const double d = E[(int64_t)a * kp + b] - (a == b ? 1.0 : 0.0);
      E[(int64_t)a * kp + b] = d;
      err += d * d;
    }
    err = block_sum<kRefThreads>(err, red);  // barrier: E complete
    if (!(err == err)) break;
    // |E|_F <= 1e-10, or no longer shrinking below 1e-9: one more step, then stop
    if (extra < 0 && (err <= 1e-20 || (err < 1e-18 && err > 0.25 * prev))) extra = 1;
    prev = err;
    ref_mm(Z, kp, false, E, kp, T, kp, n, sa, sb);    // F = Z E
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int a = e / n, b = e - a * n;
      Z[(int64_t)a * kp + b] -= 0.25 * (T[(int64_t)a * kp + b] + T[(int64_t)b * kp + a]);
    }
    __syncthreads();
    if (extra > 0 && --extra == 0) {
      ok = true;
      break;
    }
  }
  if (threadIdx.x == 0) {
    p.scal[(int64_t)i * 8 + 1] = ok ? 1.0 : 0.0;
    p.scal[(int64_t)i * 8 + 2] = (double)step;
    if (warn && !ok) raise_warning(p.status, SRM_WARN_POLAR_CONDITION);
  }
}

}  // namespace

cudaError_t launch_ns_refine(const DevPlan& p, cudaStream_t s, int warn) {
  const int n = (int)p.K;
  const size_t bytes = (size_t)2 * n * (n + 1) * sizeof(double);
  if (bytes > 227 * 1024) return cudaErrorInvalidValue;
  static size_t configured = 0;
  if (configured < bytes) {
    cudaError_t e = cudaFuncSetAttribute(k_ns_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured = bytes;
  }
  k_ns_refine<<<p.nsub, kRefThreads, bytes, s>>>(p, warn);
  return cudaGetLastError();
}

bool ns_polar_supported(int kp) { return kp >= 8 && kp <= 80 && kp % 8 == 0; }

bool ns_polar_f32_supported(int kp) { return kp > 80 && kp <= 112; }

bool ns_polar_g_supported(int kp) { return kp > 80 && kp <= 128 && kp % 8 == 0; }

cudaError_t launch_ns_polar_g(const DevPlan& p, int init, cudaStream_t s) {
  switch ((int)p.kp) {
    case 88: return run_ns_g<88>(p, init, s);
    case 96: return run_ns_g<96>(p, init, s);
    case 104: return run_ns_g<104>(p, init, s);
    case 112: return run_ns_g<112>(p, init, s);
    case 120: return run_ns_g<120>(p, init, s);
    case 128: return run_ns_g<128>(p, init, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ns_polar_f32(const DevPlan& p, int init, cudaStream_t s) {
  switch (((int)p.kp + 15) / 16 * 16) {
    case 96: return run_ns_f32<96>(p, init, s);
    case 112: return run_ns_f32<112>(p, init, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ns_polar(const DevPlan& p, int init, cudaStream_t s) {
  switch ((int)p.kp) {
    case 8: return run_ns<8>(p, init, s);
    case 16: return run_ns<16>(p, init, s);
    case 24: return run_ns<24>(p, init, s);
    case 32: return run_ns<32>(p, init, s);
    case 40: return run_ns<40>(p, init, s);
    case 48: return run_ns<48>(p, init, s);
    case 56: return run_ns<56>(p, init, s);
    case 64: return run_ns<64>(p, init, s);
    case 72: return run_ns<72>(p, init, s);
    case 80: return run_ns<80>(p, init, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace srm
