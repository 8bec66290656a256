// Probe: tcgen05.mma.cta_group::2.kind::i8 on a CTA pair (cluster of two),
// M = 256, N = 128, K = 128, SWIZZLE_128B K-major operands.  Checks which
// shared-memory rows each CTA must provide: hypothesis H1 = CTA r holds A rows
// [128 r, 128 r + 128) and B rows [64 r, 64 r + 64) at the same offsets, the
// leader (rank 0) issues the MMA and multicasts the commit; each CTA's TMEM
// lanes hold its own 128 output rows.  Rows 64..127 of each CTA's B region
// hold a junk pattern so a "B from the leader only" layout (H2) shows up too.
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

__host__ __device__ constexpr uint32_t idesc_s8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ int sw128_off(int r, int kbyte) {
  const int c = kbyte >> 4;
  return r * 128 + ((c ^ (r & 7)) << 4) + (kbyte & 15);
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// A [256][128], B [128][128] (row n = column n of the product), J [2][64][128] junk
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(const int8_t* A, const int8_t* B, const int8_t* J, int32_t* D) {
  constexpr int K = 128;
  extern __shared__ __align__(1024) int8_t dyn[];
  int8_t* base = reinterpret_cast<int8_t*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~(uintptr_t)1023);
  int8_t* sa = base;             // 128 rows
  int8_t* sb = base + 128 * K;   // 128 rows (64 own B rows + 64 junk)
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_rank();
  for (int e = tid; e < 128 * K; e += blockDim.x) sa[sw128_off(e / K, e % K)] = A[(rank * 128 + e / K) * K + e % K];
  for (int e = tid; e < 64 * K; e += blockDim.x) {
    sb[sw128_off(e / K, e % K)] = B[(rank * 64 + e / K) * K + e % K];
    sb[sw128_off(64 + e / K, e % K)] = J[(rank * 64 + e / K) * K + e % K];
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (rank == 0 && tid == 0) {
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t da = desc_sw128(smem_u32(sa) + ks * 32);
      const uint64_t db = desc_sw128(smem_u32(sb) + ks * 32);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(idesc_s8(256, 128)), "r"(ks));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&mbar)), "h"((uint16_t)3));
  }
  uint32_t done = 0;
  long spins = 0;
  while (!done && spins < 100000000) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    ++spins;
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid >> 5, lane = tid & 31, row = warp * 32 + lane;
  for (int c0 = 0; c0 < 128; c0 += 16) {
    uint32_t r[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[(rank * 128 + row) * 128 + c0 + j] = done ? (int32_t)r[j] : -999999;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  constexpr int M = 256, N = 128, K = 128;
  std::vector<int8_t> A(M * K), B(N * K), J(N * K);
  std::vector<int32_t> D(M * N);
  srand(5);
  for (auto& x : A) x = (int8_t)(rand() % 129 - 64);
  for (auto& x : B) x = (int8_t)(rand() % 129 - 64);
  for (auto& x : J) x = (int8_t)(rand() % 129 - 64);
  int8_t *dA, *dB, *dJ;
  int32_t* dD;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dJ, J.size()));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dJ, J.data(), J.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, D.size() * 4));
  const int bytes = 256 * K + 2048;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  probe<<<2, 128, bytes>>>(dA, dB, dJ, dD);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  // H1: B row n from CTA n / 64's own rows; H2: the leader's 128 B rows (B 0..63, junk 0..63)
  long bad1 = 0, bad2 = 0, timeouts = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      int32_t h1 = 0, h2 = 0;
      for (int k = 0; k < K; ++k) {
        h1 += (int32_t)A[m * K + k] * (int32_t)B[n * K + k];
        const int8_t b2 = n < 64 ? B[n * K + k] : J[(n - 64) * K + k];
        h2 += (int32_t)A[m * K + k] * (int32_t)b2;
      }
      const int32_t d = D[m * N + n];
      if (d == -999999) ++timeouts;
      if (d != h1) ++bad1;
      if (d != h2) ++bad2;
    }
  printf("cta_group::2 i8 M=256 N=128: H1 mismatches %ld, H2 mismatches %ld of %d (timeouts %ld); D[0]=%d D[200*128+100]=%d\n",
         bad1, bad2, M * N, timeouts, D[0], D[200 * 128 + 100]);
  return bad1 == 0 ? 0 : 1;
}
