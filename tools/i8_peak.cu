// Microbenchmark: dense int8 tensor-core throughput on this B200
// (tcgen05.mma kind::i8, s8 x s8 -> s32, operands resident in shared memory,
// no loads in the loop).  The measured peak is the roofline denominator of
// the int8-sliced Gram kernel (bench.py reads profiles/i8_peak.json).
//
//   1sm_128x128: cta_group::1, M = 128, N = 128 (the k_oz_gram shape)
//   1sm_128x256: cta_group::1, M = 128, N = 256
//   2sm_256x256: cta_group::2 across a CTA pair, M = 256, N = 256
//
// One CTA (or CTA pair) per SM pair, every SM busy; CUDA events around the
// launch.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_peak tools/i8_peak.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);              \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ unsigned long long g_clk[2];  // CTA 0: SM cycles and globaltimer ns of its MMA loop

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;
  return d;
}

// BL = 0: both operands K-major SW128; BL = 1: B K-major SWIZZLE_32B (rows of
// 32 B, one K step per N x 32 B block: the k_oz_sg_sk / k_oz_rowgemm B);
// BL = 2: additionally A MN-major SWIZZLE_32B (the k_oz_rowgemm<kRowW> A)
template <int CG, int M, int N, int NST, int SW = 0, int BL = 0>
__global__ void __launch_bounds__(128, 1) peak(int iters, unsigned long long seed) {
  // per CTA and stage: A 128 rows x 128 B, B (N / CG) rows x 128 B, SW128 K-major;
  // NST stages cycled (NST = 1: the same operands every MMA)
  constexpr int kRowsB = N / CG;
  constexpr int kStage = (128 + kRowsB) * 128;
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  // random operands (data-dependent power is part of the real workload)
  unsigned long long x = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * 128 + tid + 1));
  for (int e = tid; e < NST * kStage / 8; e += blockDim.x) {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    reinterpret_cast<unsigned long long*>(sm)[e] = x & 0x3F3F3F3F3F3F3F3Full;  // |q| <= 63
  }
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (tid < 32) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  constexpr uint32_t idesc = idesc_i8(M, N) | (BL == 2 ? (1u << 15) : 0u);
  const unsigned long long c0 = clock64(), g0 = gtimer();
  if (tid == 0 && rank == 0) {
    for (int it = 0; it < iters; ++it) {
      const uint32_t sa = smem_u32(sm) + (uint32_t)((it % NST) * kStage), sb = sa + 128 * 128;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t da = BL == 2 ? desc_sw32(sa + 4096 * k, 256, 1024) : desc_sw128(sa + 32 * k);
        const uint64_t db = BL >= 1 ? desc_sw32(sb + (N / CG) * 32 * k, 16, 256) : desc_sw128(sb + 32 * k);
        // SW = 0: one accumulator per 4-MMA group (alternating); SW = 1: four
        // accumulators round-robin, a switch after every MMA (the k_oz_gram d-groups)
        const uint32_t acc = SW ? tmem + (uint32_t)(k * N) % 512u : tmem + (uint32_t)((it & 1) * (N <= 256 ? N : 0)) % 512u;
        const uint32_t en = (SW ? it : (it | k)) ? 1u : 0u;
        if (CG == 1)
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(acc),
              "l"(da), "l"(db), "r"(idesc), "r"(en));
        else
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(acc),
              "l"(da), "l"(db), "r"(idesc), "r"(en));
      }
    }
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    else
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"((uint16_t)3));
  }
  if (tid == 0) {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(smem_u32(&bar)), "r"(0));
    if (blockIdx.x == 0) {
      g_clk[0] = clock64() - c0;
      g_clk[1] = gtimer() - g0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
  }
  if (tid < 32) {
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

static double g_mhz = 0.0;  // effective SM clock of the last run (CTA 0)

template <int CG, int M, int N, int NST = 1, int SW = 0, int BL = 0>
double run(int sms, int iters, int reps = 5) {
  const size_t smem = (size_t)NST * (128 + N / CG) * 128 + 1024;
  CK(cudaFuncSetAttribute(peak<CG, M, N, NST, SW, BL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms / CG * CG);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int w = 0; w < 2; ++w) CK(cudaLaunchKernelEx(&cfg, peak<CG, M, N, NST, SW, BL>, iters / 8, 7ull));
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int rep = 0; rep < reps; ++rep) {
    CK(cudaEventRecord(a));
    CK(cudaLaunchKernelEx(&cfg, peak<CG, M, N, NST, SW, BL>, iters, 11ull + rep));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  unsigned long long clk[2];
  CK(cudaMemcpyFromSymbol(clk, g_clk, sizeof(clk)));
  g_mhz = clk[1] ? (double)clk[0] / (double)clk[1] * 1e3 : 0.0;
  const double ops = 2.0 * M * N * 32.0 * 4.0 * iters * (double)(sms / CG);
  return ops / (best * 1e-3) / 1e12;
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int iters = argc > 1 ? atoi(argv[1]) : 8192;
  const double a = run<1, 128, 128>(sms, iters);
  const double b = run<1, 128, 256>(sms, iters);
  const double c = run<2, 256, 256>(sms, iters);
  const double ar = run<1, 128, 128, 6>(sms, iters);
  const double br = run<1, 128, 256, 4>(sms, iters);
  const double cr = run<2, 256, 256, 6>(sms, iters);
  const double asw = run<1, 128, 128, 6, 1>(sms, iters);
  const double n64 = run<1, 128, 64, 6>(sms, iters);
  const double n32 = run<1, 128, 32, 6>(sms, iters);
  const double burst_mhz = g_mhz;
  const double bsw32 = run<1, 128, 128, 6, 1, 1>(sms, iters);
  const double bsw32_64 = run<1, 128, 64, 6, 1, 1>(sms, iters);
  const double absw32 = run<1, 128, 128, 6, 1, 2>(sms, iters);
  // sustained: ~0.3 s of back-to-back MMAs (the clock the power controller
  // settles at under a long int8 load, as inside the Gram precompute)
  const double sus = run<1, 128, 128, 6>(sms, iters * 256, 2);
  const double sus_mhz = g_mhz;
  printf("{\"sms\": %d, \"iters\": %d, \"tops_1sm_128x128\": %.1f, \"tops_1sm_128x256\": %.1f, "
         "\"tops_2sm_256x256\": %.1f, \"tops_1sm_128x128_rot6\": %.1f, \"tops_1sm_128x256_rot4\": %.1f, "
         "\"tops_2sm_256x256_rot6\": %.1f, \"tops_1sm_128x128_rot6_accswitch\": %.1f, \"burst_sm_mhz\": %.0f, "
         "\"tops_1sm_128x128_sustained\": %.1f, \"sustained_sm_mhz\": %.0f, \"tops_1sm_128x64_rot6\": %.1f, "
         "\"tops_1sm_128x32_rot6\": %.1f, \"tops_128x128_accswitch_b_sw32\": %.1f, "
         "\"tops_128x64_accswitch_b_sw32\": %.1f, \"tops_128x128_accswitch_a_mn_sw32_b_sw32\": %.1f}\n",
         sms, iters, a, b, c, ar, br, cr, asw, burst_mhz, sus, sus_mhz, n64, n32, bsw32, bsw32_64, absw32);
  return 0;
}
