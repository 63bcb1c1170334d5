// Layout check: tcgen05.mma kind::tf32 with the A operand in tensor memory (M = 128 rows on the
// 128 TMEM lanes, K along 32-bit columns), written by tcgen05.st from registers as the exact tf32
// pair a = hi + lo; B (N × 32, K-major SWIZZLE_128B) in shared memory.  3xTF32 product
// lo·hi + hi·lo + hi·hi into one accumulator, compared with the fp64 product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_00420_b200/csrc -o tools/ts_mma_test tools/ts_mma_test.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "umma.cuh"

using namespace cmtcs::umma;

constexpr int M = 128, K = 32, NB = 80;

__device__ __forceinline__ float rna(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float *v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}

__global__ void k(const float *A, const float *B, float *C) {
  __shared__ __align__(1024) unsigned char bs[2 * NB * 128];
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, w = t >> 5;
  // B hi / lo tiles, SW128 K-major
  for (int e = t; e < NB * K; e += 128) {
    const int n = e / K, kk = e % K;
    const float x = B[e], h = rna(x);
    const uint32_t off = sw128_offset(n, kk / 4) + (kk % 4) * 4;
    *reinterpret_cast<float *>(bs + off) = h;
    *reinterpret_cast<float *>(bs + NB * 128 + off) = x - h;
  }
  if (t == 0) mbar_init(&done, 1);
  if (w == 0) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = slot;
  // A row t (lane t): hi at columns [256, 288), lo at [288, 320)
  {
    float h[16], l[16];
    for (int half = 0; half < 2; ++half) {
      for (int i = 0; i < 16; ++i) {
        const float x = A[t * K + 16 * half + i];
        h[i] = rna(x);
        l[i] = x - h[i];
      }
      const uint32_t lane_addr = tm + ((uint32_t)(w * 32) << 16);
      tmem_st16(lane_addr + 256 + 16 * half, h);
      tmem_st16(lane_addr + 288 + 16 * half, l);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (t == 0) {
    const uint32_t idesc = idesc_tf32(M, NB);
    const uint64_t bh = desc_sw128(smem_u32(bs)), bl = desc_sw128(smem_u32(bs + NB * 128));
    for (int k8 = 0; k8 < K / 8; ++k8) {
      const uint64_t o = (uint64_t)(k8 * 32) >> 4;
      mma_ts(tm, tm + 288 + 8 * k8, bh + o, idesc, k8 > 0);   // lo · hi
      mma_ts(tm, tm + 256 + 8 * k8, bl + o, idesc, 1);        // hi · lo
      mma_ts(tm, tm + 256 + 8 * k8, bh + o, idesc, 1);        // hi · hi
    }
    mma_commit(&done);
  }
  mbar_wait(&done, 0);
  fence_after_sync();
  float v[16];
  for (int c0 = 0; c0 < NB; c0 += 16) {
    tmem_ld16(tm + ((uint32_t)(w * 32) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) C[t * NB + c0 + i] = v[i];
  }
  fence_before_sync();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tm);
}

int main() {
  float *hA = new float[M * K], *hB = new float[NB * K], *hC = new float[M * NB];
  srand(7);
  for (int i = 0; i < M * K; ++i) hA[i] = (float)rand() / RAND_MAX * 2 - 1;
  for (int i = 0; i < NB * K; ++i) hB[i] = (float)rand() / RAND_MAX * 2 - 1;
  float *A, *B, *C;
  cudaMalloc(&A, M * K * 4);
  cudaMalloc(&B, NB * K * 4);
  cudaMalloc(&C, M * NB * 4);
  cudaMemcpy(A, hA, M * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, NB * K * 4, cudaMemcpyHostToDevice);
  k<<<1, 128>>>(A, B, C);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hC, C, M * NB * 4, cudaMemcpyDeviceToHost);
  double maxrel = 0, maxabs = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NB; ++n) {
      double s = 0, sa = 0;
      for (int kk = 0; kk < K; ++kk) { s += (double)hA[m * K + kk] * hB[n * K + kk]; sa += fabs((double)hA[m * K + kk] * hB[n * K + kk]); }
      const double d = fabs(hC[m * NB + n] - s);
      maxabs = d > maxabs ? d : maxabs;
      maxrel = d / sa > maxrel ? d / sa : maxrel;
    }
  printf("%s: max |err| %.3e, max |err|/sum|a b| %.3e (fp32 level ~1e-7; garbage ~1)\n", cudaGetErrorString(e), maxabs, maxrel);
  return 0;
}
