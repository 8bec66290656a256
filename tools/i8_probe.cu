// Probe: tcgen05.mma kind::i8 (s8 x s8 -> s32) with SWIZZLE_128B K-major smem
// operands and a TMEM accumulator.  Validates the instruction-descriptor and
// smem-descriptor encodings of the int8 Gram kernel (exact integer results).
// Single CTA, M = 128, N = NN, K = 128 (four K = 32 steps).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, uint32_t dfmt, uint32_t afmt) {
  return (dfmt << 4) | (afmt << 7) | (afmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// row r (128 B of K) of a K-major SW128 tile: 16-byte chunk c lives at chunk c ^ (r & 7)
__device__ __forceinline__ int sw128_off(int r, int kbyte) {
  const int c = kbyte >> 4;
  return r * 128 + ((c ^ (r & 7)) << 4) + (kbyte & 15);
}

template <int NN>
__global__ void probe(const int8_t* A, const int8_t* B, int32_t* D, uint32_t idesc) {
  constexpr int M = 128, K = 128;
  extern __shared__ __align__(1024) int8_t dyn[];
  int8_t* sa = dyn;
  int8_t* sb = dyn + M * K;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  for (int e = tid; e < M * K; e += blockDim.x) sa[sw128_off(e / K, e % K)] = A[e];
  for (int e = tid; e < NN * K; e += blockDim.x) sb[sw128_off(e / K, e % K)] = B[e];
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t da = desc_sw128(smem_u32(sa) + ks * 32);
      const uint64_t db = desc_sw128(smem_u32(sb) + ks * 32);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(idesc), "r"(ks));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid >> 5, lane = tid & 31, row = warp * 32 + lane;
  for (int c0 = 0; c0 < NN; c0 += 16) {
    uint32_t r[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[row * NN + c0 + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int NN>
void run(uint32_t dfmt, uint32_t afmt, int lim) {
  constexpr int M = 128, K = 128;
  std::vector<int8_t> A(M * K), B(NN * K);
  std::vector<int32_t> D(M * NN);
  srand(11);
  for (auto& x : A) x = (int8_t)(rand() % (2 * lim + 1) - lim);
  for (auto& x : B) x = (int8_t)(rand() % (2 * lim + 1) - lim);
  int8_t *dA, *dB;
  int32_t* dD;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, D.size() * 4));
  const int bytes = (M + NN) * K + 1024;
  CK(cudaFuncSetAttribute(probe<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  probe<NN><<<1, 128, bytes>>>(dA, dB, dD, idesc_i8(M, NN, dfmt, afmt));
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NN; ++n) {
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += (int32_t)A[m * K + k] * (int32_t)B[n * K + k];
      if (ref != D[m * NN + n]) ++bad;
    }
  int32_t r00 = 0;
  for (int k = 0; k < K; ++k) r00 += (int32_t)A[k] * (int32_t)B[k];
  printf("i8 N=%d dfmt=%u afmt=%u lim=%d: mismatches %ld / %d  D[0]=%d ref %d\n", NN, dfmt, afmt, lim, bad, M * NN, D[0], r00);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

// B operand MN-major: smem rows are K (128 of them), each 128 bytes of N, SW128;
// MN blocks of 128 bytes are KB * 128 bytes apart (LBO); 8-row groups 1024 B (SBO)
template <int NN>
__global__ void probe_mn(const int8_t* A, const int8_t* B, int32_t* D, uint32_t idesc, int lbo_mode) {
  constexpr int M = 128, K = 128;
  extern __shared__ __align__(1024) int8_t dyn[];
  int8_t* sa = dyn;
  int8_t* sb = dyn + M * K;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  for (int e = tid; e < M * K; e += blockDim.x) sa[sw128_off(e / K, e % K)] = A[e];
  // B logical [n][k]; stored: block nb = n / 128, row k, byte n % 128
  for (int e = tid; e < NN * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    sb[(n >> 7) * (K * 128) + sw128_off(k, n & 127)] = B[e];
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t da = desc_sw128(smem_u32(sa) + ks * 32);
      uint64_t db = desc_sw128(smem_u32(sb) + ks * 32 * 128);
      const uint32_t lbo = lbo_mode == 0 ? K * 128 : (lbo_mode == 1 ? 1024 : 128);
      db = (db & ~(((uint64_t)0x3FFF) << 16)) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(idesc), "r"(ks));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid >> 5, lane = tid & 31, row = warp * 32 + lane;
  for (int c0 = 0; c0 < NN; c0 += 16) {
    uint32_t r[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[row * NN + c0 + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int NN>
void run_mn(int lbo_mode) {
  constexpr int M = 128, K = 128;
  std::vector<int8_t> A(M * K), B(NN * K);
  std::vector<int32_t> D(M * NN);
  srand(13);
  for (auto& x : A) x = (int8_t)(rand() % 129 - 64);
  for (auto& x : B) x = (int8_t)(rand() % 129 - 64);
  int8_t *dA, *dB;
  int32_t* dD;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, D.size() * 4));
  const int bytes = (M + NN) * K + 1024;
  CK(cudaFuncSetAttribute(probe_mn<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  const uint32_t idesc = idesc_i8(M, NN, 2, 1) | (1u << 16);  // B MN-major
  probe_mn<NN><<<1, 128, bytes>>>(dA, dB, dD, idesc, lbo_mode);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NN; ++n) {
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += (int32_t)A[m * K + k] * (int32_t)B[n * K + k];
      if (ref != D[m * NN + n]) ++bad;
    }
  printf("i8 B MN-major N=%d lbo_mode=%d: mismatches %ld / %d\n", NN, lbo_mode, bad, M * NN);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
}


// A operand MN-major, SWIZZLE_32B: smem = [mblk (M/32)][k rows (K)][32 bytes of m],
// each 8-row group a 256-byte swizzle atom; LBO = distance between m-blocks
// (K * 32 bytes), SBO = 8 rows * 32 B = 256.  TMA SWIZZLE_32B layout within an
// atom: the 16-byte chunk c (0..1) of row r lives at chunk c ^ ((r >> 2) & 1).
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;  // SWIZZLE_32B
  return d;
}

__global__ void probe_amn(const int8_t* A, const int8_t* B, int32_t* D, uint32_t idesc, int swz_mode) {
  constexpr int M = 128, K = 128, NN = 64;
  extern __shared__ __align__(1024) int8_t dyn[];
  int8_t* sa = dyn;
  int8_t* sb = dyn + M * K;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  // A logical [m][k]: block mb = m / 32, row k, byte m % 32 (chunk swizzle per swz_mode)
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    const int mb = m >> 5, mc = m & 31;
    int chunk = mc >> 4;
    if (swz_mode == 1) chunk ^= (k >> 2) & 1;
    if (swz_mode == 2) chunk ^= (k >> 3) & 1;
    if (swz_mode == 3) chunk ^= k & 1;
    sa[mb * (K * 32) + k * 32 + chunk * 16 + (mc & 15)] = A[e];
  }
  for (int e = tid; e < NN * K; e += blockDim.x) sb[sw128_off(e / K, e % K)] = B[e];
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t da = desc_sw32(smem_u32(sa) + ks * 32 * 32, K * 32, 256);
      const uint64_t db = desc_sw128(smem_u32(sb) + ks * 32);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(idesc), "r"(ks));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid >> 5, lane = tid & 31, row = warp * 32 + lane;
  for (int c0 = 0; c0 < NN; c0 += 16) {
    uint32_t r[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[row * NN + c0 + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

void run_amn(int swz_mode) {
  constexpr int M = 128, K = 128, NN = 64;
  std::vector<int8_t> A(M * K), B(NN * K);
  std::vector<int32_t> D(M * NN);
  srand(17);
  for (auto& x : A) x = (int8_t)(rand() % 129 - 64);
  for (auto& x : B) x = (int8_t)(rand() % 129 - 64);
  int8_t *dA, *dB;
  int32_t* dD;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, D.size() * 4));
  const int bytes = (M + NN) * K + 1024;
  CK(cudaFuncSetAttribute(probe_amn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  const uint32_t idesc = idesc_i8(M, NN, 2, 1) | (1u << 15);  // A MN-major
  probe_amn<<<1, 128, bytes>>>(dA, dB, dD, idesc, swz_mode);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NN; ++n) {
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += (int32_t)A[m * K + k] * (int32_t)B[n * K + k];
      if (ref != D[m * NN + n]) ++bad;
    }
  printf("i8 A MN-major SW32 swz_mode=%d: mismatches %ld / %d\n", swz_mode, bad, M * NN);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

int main() {
  for (int m = 0; m < 4; ++m) run_amn(m);
  run<128>(2, 1, 64);
  run<256>(2, 1, 64);
  run<256>(2, 1, 127);
  run<64>(2, 1, 127);
  for (int mode = 0; mode < 3; ++mode) {
    run_mn<128>(mode);
    run_mn<256>(mode);
  }
  return 0;
}
