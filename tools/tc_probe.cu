// Probe: tcgen05.mma kind::tf32 with K-major / MN-major SWIZZLE_NONE smem
// descriptors, TMEM accumulator, 3xTF32 split precision.  Validates the
// descriptor encodings used by the fp32 streaming kernels against fp64 on the
// host.  Single CTA, M = 128, N = NN, K = 32.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// MODE 0: A K-major (M x K, K contiguous in global), B K-major (N x K)   [A-pass shape]
// MODE 1: A MN-major (K x M, M contiguous in global), B MN-major (K x N) [B-pass shape]
template <int NN, int MODE>
__global__ void probe(const float* A, const float* B, float* D, int amn, int bmn, int var) {
  constexpr int M = 128, K = 32;
  extern __shared__ __align__(1024) float dyn[];
  float* sa_hi = dyn;
  float* sa_lo = sa_hi + M * K;
  float* sb_hi = sa_lo + M * K;
  float* sb_lo = sb_hi + NN * K;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  // canonical SWIZZLE_NONE core-matrix layouts (element offsets)
  auto kmaj = [](int mn, int k, int mnsize) {  // core = 8 MN rows x 4 K (16 B), LBO=128B (K), SBO=(K/4)*128B (MN)
    return (mn >> 3) * (K / 4) * 32 + (k >> 2) * 32 + (mn & 7) * 4 + (k & 3);
  };
  auto kmaj2 = [](int mn, int k, int mnsize) {  // MN-major alt: core = 8 MN (32 B?) no: 8 K rows of 16B MN, cores along K first
    return (mn >> 2) * (K / 8) * 32 + (k >> 3) * 32 + (k & 7) * 4 + (mn & 3);
  };
  auto mnmaj = [](int mn, int k, int mnsize) {  // core = 4 MN (16 B) x 8 K rows; SBO=128B (MN), LBO=(MN/4)*128B (K)
    return (k >> 3) * (mnsize / 4) * 32 + (mn >> 2) * 32 + (k & 7) * 4 + (mn & 3);
  };
  for (int e = tid; e < M * K; e += blockDim.x) {
    int m, k;
    float x;
    m = e / K; k = e % K; x = A[m * K + k];
    const int o = amn == 0 ? kmaj(m, k, M) : (var == 2 ? kmaj2(m, k, M) : mnmaj(m, k, M));
    const float h = tf32_hi(x);
    sa_hi[o] = h;
    sa_lo[o] = x - h;
  }
  for (int e = tid; e < NN * K; e += blockDim.x) {
    int n, k;
    float x;
    n = e / K; k = e % K; x = B[n * K + k];
    const int o = bmn == 0 ? kmaj(n, k, NN) : (var == 2 ? kmaj2(n, k, NN) : mnmaj(n, k, NN));
    const float h = tf32_hi(x);
    sb_hi[o] = h;
    sb_lo[o] = x - h;
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, NN, amn, bmn);
    for (int ks = 0; ks < K / 8; ++ks) {
      uint64_t dah, dal, dbh, dbl;
      auto mk = [&](float* base, int mn, int size) -> uint64_t {
        if (!mn) return sdesc(smem_u32(base) + ks * 256, 128, (K / 4) * 128);
        if (var == 0) return sdesc(smem_u32(base) + ks * (size / 4) * 128, (size / 4) * 128, 128);
        if (var == 1) return sdesc(smem_u32(base) + ks * (size / 4) * 128, 128, (size / 4) * 128);
        return sdesc(smem_u32(base) + ks * 128, 128, (K / 8) * 128);  // var 2: kmaj2 layout
      };
      dah = mk(sa_hi, amn, M); dal = mk(sa_lo, amn, M);
      dbh = mk(sb_hi, bmn, NN); dbl = mk(sb_lo, bmn, NN);
      mma_tf32(tmem, dah, dbh, id, ks > 0);
      mma_tf32(tmem, dah, dbl, id, 1);
      mma_tf32(tmem, dal, dbh, id, 1);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  // wait for the MMAs (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid >> 5, lane = tid & 31;
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < NN; c0 += 16) {
    uint32_t r[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[row * NN + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(256));
}

template <int NN, int MODE>
void run(int amn, int bmn, int var) {
  constexpr int M = 128, K = 32;
  std::vector<float> A(M * K), B(NN * K), D(M * NN);
  srand(7 + MODE);
  for (auto& x : A) x = (float)rand() / RAND_MAX * 2 - 1;
  for (auto& x : B) x = (float)rand() / RAND_MAX * 2 - 1;
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, D.size() * 4));
  const int bytes = (2 * M * K + 2 * NN * K) * 4;
  CK(cudaFuncSetAttribute(probe<NN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  probe<NN, MODE><<<1, 128, bytes>>>(dA, dB, dD, amn, bmn, var);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NN; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) {
        const double a = A[m * K + k];
        const double b = B[n * K + k];
        ref += a * b;
      }
      maxerr = fmax(maxerr, fabs(ref - D[m * NN + n]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("amn %d bmn %d var %d N=%d: max abs err %.3e (max |ref| %.3f) -> rel %.3e  D[0]=%f D[1]=%f\n", amn, bmn, var, NN, maxerr, maxref,
         maxerr / maxref, D[0], D[1]); (void)MODE; (void)amn;
}


// A operand from TMEM: lane = row m, 32-bit column = k.  raw at cols [128,160), lo at [160,192)
__global__ void probe_ts(const float* A, const float* B, float* D) {
  constexpr int M = 128, K = 32, NN = 112;
  extern __shared__ __align__(1024) float dyn[];
  float* sb_hi = dyn;
  float* sb_lo = sb_hi + NN * K;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto kmaj = [](int mn, int k) { return (mn >> 3) * (K / 4) * 32 + (k >> 2) * 32 + (mn & 7) * 4 + (k & 3); };
  for (int e = tid; e < NN * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    const float x = B[n * K + k];
    const float h = tf32_hi(x);
    sb_hi[kmaj(n, k)] = h;
    sb_lo[kmaj(n, k)] = x - h;
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  // each thread stores its row: raw (32 cols) and lo (32 cols)
  {
    const int row = warp * 32 + lane;
    uint32_t raw[32], lo[32];
    for (int k = 0; k < K; ++k) {
      const float x = A[row * K + k];
      raw[k] = __float_as_uint(x);
      lo[k] = __float_as_uint(x - tf32_hi(x));
    }
    const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 32; c += 16) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                   :: "r"(base + 128 + c), "r"(raw[c]), "r"(raw[c+1]), "r"(raw[c+2]), "r"(raw[c+3]), "r"(raw[c+4]), "r"(raw[c+5]), "r"(raw[c+6]), "r"(raw[c+7]),
                      "r"(raw[c+8]), "r"(raw[c+9]), "r"(raw[c+10]), "r"(raw[c+11]), "r"(raw[c+12]), "r"(raw[c+13]), "r"(raw[c+14]), "r"(raw[c+15]));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                   :: "r"(base + 160 + c), "r"(lo[c]), "r"(lo[c+1]), "r"(lo[c+2]), "r"(lo[c+3]), "r"(lo[c+4]), "r"(lo[c+5]), "r"(lo[c+6]), "r"(lo[c+7]),
                      "r"(lo[c+8]), "r"(lo[c+9]), "r"(lo[c+10]), "r"(lo[c+11]), "r"(lo[c+12]), "r"(lo[c+13]), "r"(lo[c+14]), "r"(lo[c+15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t id = idesc_tf32(M, NN, 0, 0);
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t dbh = sdesc(smem_u32(sb_hi) + ks * 256, 128, (K / 4) * 128);
      const uint64_t dbl = sdesc(smem_u32(sb_lo) + ks * 256, 128, (K / 4) * 128);
      const uint32_t ar = tmem + 128 + ks * 8, al = tmem + 160 + ks * 8;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                   :: "r"(tmem), "r"(ar), "l"(dbh), "r"(id), "r"(ks > 0 ? 1 : 0));
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                   :: "r"(tmem), "r"(ar), "l"(dbl), "r"(id), "r"(1));
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                   :: "r"(tmem), "r"(al), "l"(dbh), "r"(id), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < NN; c0 += 16) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[row * NN + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(256));
}

void run_ts() {
  constexpr int M = 128, K = 32, NN = 112;
  std::vector<float> A(M * K), B(NN * K), D(M * NN);
  srand(11);
  for (auto& x : A) x = (float)rand() / RAND_MAX * 2 - 1;
  for (auto& x : B) x = (float)rand() / RAND_MAX * 2 - 1;
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, D.size() * 4));
  const int bytes = 2 * NN * K * 4;
  probe_ts<<<1, 128, bytes>>>(dA, dB, dD);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NN; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - D[m * NN + n]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("TS (A in TMEM) N=%d: rel err %.3e  D[0]=%f\n", NN, maxerr / maxref, D[0]);
}

int main() {
  run_ts();
  for (int var = 0; var < 3; ++var) {
    run<64, 0>(1, 0, var);
    run<64, 0>(0, 1, var);
    run<64, 0>(1, 1, var);
  }
  run<64, 0>(0, 0, 0);
  return 0;
}
