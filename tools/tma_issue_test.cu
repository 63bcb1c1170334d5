// Microbenchmark: TMA issue cost of the CG kernel's producer pattern — per ring stage one
// arrive.expect_tx and NB 2-D tile loads (16 KB A box + B boxes) from an L2-resident source, a
// 4-stage ring released immediately by a consumer warp.  Variants: single-lane producer vs a
// converged warp issuing through elect.sync.  Cycles per stage on the producer (clock64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_issue_test tools/tma_issue_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t *m, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(m)), "r"(c) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(m)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *m, uint32_t ph) {
  asm volatile("{\n\t.reg .pred done;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t@!done bra W_%=;\n\t}\n" ::"r"(su32(m)), "r"(ph) : "memory");
}
template <bool WARP>
__device__ __forceinline__ void arrive_tx(uint64_t *m, uint32_t b) {
  if (WARP)
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}\n" ::"r"(su32(m)), "r"(b) : "memory");
  else
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(m)), "r"(b) : "memory");
}
template <bool WARP>
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *mb) {
  if (WARP)
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n\t}\n" ::"r"(su32(dst)),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(mb)) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(su32(dst)),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(mb)) : "memory");
}

constexpr int S = 4, STAGE = 48 * 1024;

template <bool WARP, int NB>
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                             int chunks, unsigned long long *out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S], empty[S];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { init(&full[s], 1); init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const uint32_t bytes = 16384 + (NB - 1) * 10240;
  if (warp == 0 && (WARP || lane == 0)) {
    const long long c0 = clock64();
    int st = 0; uint32_t ph = 0;
    for (int g = 0; g < chunks; ++g) {
      if (g >= S) wait(&empty[st], ph ^ 1u);
      unsigned char *base = sm + st * STAGE;
      arrive_tx<WARP>(&full[st], bytes);
      const int kk = (g & 7) * 32;
      tma2d<WARP>(base, &ma, kk, (blockIdx.x & 7) * 128, &full[st]);
      for (int b = 1; b < NB; ++b) tma2d<WARP>(base + 16384 + (b - 1) * 10240, &mb, kk, b * 80, &full[st]);
      if (++st == S) { st = 0; ph ^= 1u; }
    }
    const long long c1 = clock64();
    if (lane == 0) out[blockIdx.x] = c1 - c0;
  } else if (warp == 1) {
    int st = 0; uint32_t ph = 0;
    for (int g = 0; g < chunks; ++g) {
      wait(&full[st], ph);
      __syncwarp();
      if (lane == 0) arrive(&empty[st]);
      if (++st == S) { st = 0; ph ^= 1u; }
    }
  }
}

typedef CUresult (*Enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                        const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <bool WARP, int NB>
void run(const CUtensorMap &ma, const CUtensorMap &mb, unsigned long long *out) {
  unsigned long long h[148];
  const int chunks = 4000;
  cudaFuncSetAttribute(k<WARP, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * STAGE + 1024);
  for (int r = 0; r < 2; ++r) k<WARP, NB><<<148, 128, S * STAGE + 1024>>>(ma, mb, chunks, out);
  cudaDeviceSynchronize();
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%s producer, %d TMA loads per stage: %.0f clk per stage  (%s)\n", WARP ? "warp+elect " : "single-lane", NB,
         (double)mx / chunks, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float *a, *b;
  cudaMalloc(&a, 1024 * 256 * 4);   // 1 MB: L2-resident
  cudaMalloc(&b, 512 * 256 * 4);
  cudaMemset(a, 0, 1024 * 256 * 4);
  cudaMemset(b, 0, 512 * 256 * 4);
  unsigned long long *out;
  cudaMalloc(&out, 148 * 8);
  void *fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  CUtensorMap ma, mb;
  {
    cuuint64_t dims[2] = {256, 1024}, str[1] = {256 * 4};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[2] = {256, 512}, str[1] = {256 * 4};
    cuuint32_t box[2] = {32, 80}, es[2] = {1, 1};
    enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, b, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  run<false, 1>(ma, mb, out);
  run<false, 3>(ma, mb, out);
  run<true, 1>(ma, mb, out);
  run<true, 3>(ma, mb, out);
  return 0;
}
