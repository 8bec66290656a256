// Does a small CTA get placed on an SM that already holds one big persistent
// CTA (the int8 Gram's footprint: 320 threads x ~168 registers, ~197 KB of
// dynamic shared memory, 512 TMEM columns, high-priority stream)?
// usage: coresidency_probe <tmem 0/1> <prio 0/1> <big_regs 0..4: ~17/149/49/81/113> <big_smem_kb> <small_threads> <small_smem_kb> <big max carve-out 0/1>
// Prints how many small CTAs started while the big kernel was still running
// and on how many distinct SMs.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <set>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}

template <int REGS>
__global__ void __launch_bounds__(320, 1) k_big(int use_tmem, unsigned long long spin_ns, unsigned long long* endt, float* sink) {
  extern __shared__ unsigned char sm[];
  __shared__ unsigned tbase;
  if (use_tmem && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  float acc[REGS];
#pragma unroll
  for (int j = 0; j < REGS; ++j) acc[j] = threadIdx.x * 0.5f + j;
  const unsigned long long t0 = gtime();
  while (gtime() - t0 < spin_ns) {
#pragma unroll
    for (int j = 0; j < REGS; ++j) acc[j] = acc[j] * 1.0001f + acc[(j + 1) % REGS];
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < REGS; ++j) s += acc[j];
  sm[threadIdx.x] = (unsigned char)s;
  sink[blockIdx.x * 320 + threadIdx.x] = s + sm[(threadIdx.x + 1) % 320];
  __syncthreads();
  if (use_tmem && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  if (threadIdx.x == 0) endt[blockIdx.x] = gtime();
}

__global__ void k_small(unsigned long long* startt, unsigned* sm_of, unsigned long long hold_ns) {
  extern __shared__ unsigned char sm2[];
  if (threadIdx.x == 0) {
    startt[blockIdx.x] = gtime();
    sm_of[blockIdx.x] = smid();
    if (hold_ns == 1) sm2[0] = 1;
  }
  const unsigned long long t0 = gtime();
  while (gtime() - t0 < hold_ns) {}
}

int main(int argc, char** argv) {
  const int tmem = argc > 1 ? atoi(argv[1]) : 1, prio = argc > 2 ? atoi(argv[2]) : 1, bigregs = argc > 3 ? atoi(argv[3]) : 1;
  const int big_kb = argc > 4 ? atoi(argv[4]) : 193, sthreads = argc > 5 ? atoi(argv[5]) : 128, small_kb = argc > 6 ? atoi(argv[6]) : 9;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t sb, ss;
  cudaStreamCreateWithPriority(&sb, cudaStreamNonBlocking, prio ? hi : lo);
  cudaStreamCreateWithPriority(&ss, cudaStreamNonBlocking, lo);
  const int nbig = 144, nsmall = 4096;
  unsigned long long *endt, *startt;
  unsigned* smof;
  float* sink;
  cudaMalloc(&endt, nbig * 8);
  cudaMalloc(&startt, nsmall * 8);
  cudaMalloc(&smof, nsmall * 4);
  cudaMalloc(&sink, nbig * 320 * 4);
  const size_t big_bytes = (size_t)big_kb * 1024;
  const void* bigs[5] = {(const void*)k_big<8>, (const void*)k_big<140>, (const void*)k_big<40>, (const void*)k_big<72>,
                         (const void*)k_big<104>};
  const void* bigf = bigs[bigregs];
  cudaFuncSetAttribute(bigf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_bytes);
  if (argc > 7 && atoi(argv[7]))  // the big kernel asks for the maximum shared-memory carve-out
    cudaFuncSetAttribute(bigf, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, bigf);
  printf("big kernel regs %d, small threads %d smem %d KB, tmem %d prio %d big smem %d KB\n", fa.numRegs, sthreads, small_kb, tmem, prio, big_kb);
  for (int rep = 0; rep < 2; ++rep) {
    {
      unsigned long long spin = 1000000ull;
      void* args[] = {(void*)&tmem, (void*)&spin, (void*)&endt, (void*)&sink};
      cudaLaunchKernel(bigf, dim3(nbig), dim3(320), args, big_bytes, sb);
    }
    k_small<<<nsmall, sthreads, (size_t)small_kb * 1024, ss>>>(startt, smof, 20000ull);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  }
  std::vector<unsigned long long> he(nbig), hs(nsmall);
  std::vector<unsigned> hm(nsmall);
  cudaMemcpy(he.data(), endt, nbig * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hs.data(), startt, nsmall * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hm.data(), smof, nsmall * 4, cudaMemcpyDeviceToHost);
  unsigned long long first_end = ~0ull;
  for (auto t : he) first_end = t < first_end ? t : first_end;
  int early = 0;
  std::set<unsigned> sms;
  for (int b = 0; b < nsmall; ++b)
    if (hs[b] < first_end) { ++early; sms.insert(hm[b]); }
  printf("small CTAs started before the first big CTA ended: %d of %d, on %zu distinct SMs\n", early, nsmall, sms.size());
  return 0;
}
