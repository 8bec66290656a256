// Probe: a 5-D TMA box over the int8 Gram slice records Q[subj][t][vb][slot][32]
// with dims ordered {32 B, t, vb, slot, subj} (non-monotonic strides) and
// SWIZZLE_32B, so that one load lands as [slot][vb][t][32 B] -- per slot the
// MN-major SW32 A operand (m-blocks = voxel blocks, K rows = TRs).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int NSUB = 2, LDX = 64, NVB = 8, BOXT = 32, BOXVB = 4, BOXS = 7;
constexpr int LQ = NVB * 256;
constexpr int BYTES = 32 * BOXT * BOXVB * BOXS;

__global__ void load(const __grid_constant__ CUtensorMap tm, uint8_t* out, int t0, int vb0, int subj) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(&bar)), "r"(BYTES));
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(t0), "r"(vb0), "r"(0), "r"(subj),
        "r"(smem_u32(&bar)) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(0));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < BYTES; e += blockDim.x) out[e] = sm[e];
}

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  auto encode = reinterpret_cast<EncodeTiledFn>(fp);
  const size_t n = (size_t)NSUB * LDX * LQ;
  std::vector<uint8_t> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (uint8_t)((i * 2654435761u) >> 13);
  uint8_t *dq, *dout;
  CK(cudaMalloc(&dq, n));
  CK(cudaMalloc(&dout, BYTES));
  CK(cudaMemcpy(dq, h.data(), n, cudaMemcpyHostToDevice));
  CUtensorMap tm;
  cuuint64_t dims[5] = {32, LDX, NVB, 8, NSUB};
  cuuint64_t strides[4] = {LQ, 256, 32, (cuuint64_t)LDX * LQ};
  cuuint32_t box[5] = {32, BOXT, BOXVB, BOXS, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, dq, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode 5-D non-monotonic: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 0;
  const int t0 = 32, vb0 = 4, subj = 1;
  CK(cudaFuncSetAttribute(load, cudaFuncAttributeMaxDynamicSharedMemorySize, BYTES + 1024));
  load<<<1, 256, BYTES + 1024>>>(tm, dout, t0, vb0, subj);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<uint8_t> o(BYTES);
  CK(cudaMemcpy(o.data(), dout, BYTES, cudaMemcpyDeviceToHost));
  // expected: [slot][vb][t][32 B], 16-byte chunk c of row (t) at chunk c ^ ((t >> 2) & 1) within each 256-B atom
  long bad = 0;
  for (int s = 0; s < BOXS; ++s)
    for (int vb = 0; vb < BOXVB; ++vb)
      for (int t = 0; t < BOXT; ++t)
        for (int b = 0; b < 32; ++b) {
          const size_t src = ((size_t)subj * LDX + t0 + t) * LQ + (size_t)(vb0 + vb) * 256 + s * 32 + b;
          const int chunk = (b >> 4) ^ ((t >> 2) & 1);
          const size_t dst = (((size_t)s * BOXVB + vb) * BOXT + t) * 32 + chunk * 16 + (b & 15);
          if (o[dst] != h[src]) ++bad;
        }
  printf("5-D box layout [slot][vb][t][32 B] with SW32 chunk swizzle: mismatches %ld / %d\n", bad, BYTES);
  return 0;
}
