// Microbenchmark: DMMA.8x8x4 throughput per warp with NACC independent accumulators, with and
// without an fp32 → fp64 conversion (F2F) feeding each MMA's A operand (the mean-column pattern);
// NW warps per CTA doing it (one per SMSP when 4), 148 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_test tools/dmma_test.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double f2d_int(float x) {
  const uint32_t u = __float_as_uint(x), m = u & 0x7fffffffu, s = u & 0x80000000u;
  const uint32_t hi = m ? (s | ((m >> 3) + 0x38000000u)) : s;
  return __hiloint2double((int)hi, (int)(m << 29));
}
template <int NACC, int CVT>
__global__ void k(int iters, int nw, float *src, unsigned long long *out) {
  const int w = threadIdx.x >> 5;
  double acc[NACC][2];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  float fa[NACC];
  double da[NACC];
  for (int i = 0; i < NACC; ++i) { fa[i] = src[(threadIdx.x + i) & 255]; da[i] = fa[i]; }
  double b = src[threadIdx.x & 255];
  const long long c0 = clock64();
  if (w < nw) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) {
        const double a = CVT == 2 ? f2d_int(fa[i]) : CVT == 1 ? (double)fa[i] : da[i];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
      }
#pragma unroll
      for (int i = 0; i < NACC; ++i) fa[i] += 1.0f;
    }
  }
  const long long c1 = clock64();
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) src[0] = 0;
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
}
template <int NACC, int CVT>
void run(int nw) {
  float *src;
  unsigned long long *out, h[148];
  cudaMalloc(&src, 1024 * 4);
  cudaMemset(src, 0, 4096);
  cudaMalloc(&out, 148 * 8);
  const int iters = 2000;
  for (int r = 0; r < 2; ++r) k<NACC, CVT><<<148, 384>>>(iters, nw, src, out);
  cudaDeviceSynchronize();
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("NACC=%d cvt=%d warps=%d: %.1f clk per DMMA per warp  (%s)\n", NACC, CVT, nw, (double)h[0] / (iters * NACC),
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<1, 0>(1); run<2, 0>(1); run<1, 0>(4); run<2, 0>(4);   // NACC = 1: the dependent-chain latency
  for (int nw : {1, 4, 8}) {
    run<4, 0>(nw); run<4, 1>(nw); run<4, 2>(nw); run<8, 0>(nw); run<8, 1>(nw); run<8, 2>(nw);
  }
  return 0;
}
