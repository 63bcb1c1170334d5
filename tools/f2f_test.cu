// Microbenchmark: throughput of fp32 -> fp64 conversion (F2F.F64.F32) vs an integer bit-trick
// conversion, and of DMUL, on the B200 (148 SMs x 384 threads, 1 CTA per SM like k_cg_persistent).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/f2f_test tools/f2f_test.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double f2d_bits(float x) {
  const uint32_t u = __float_as_uint(x), mag = u & 0x7fffffffu;
  if (mag - 0x00800000u >= 0x7f000000u) return (double)x;   // zero, denormal, inf, nan
  const uint32_t hi = (u & 0x80000000u) | ((mag >> 3) + (896u << 20));
  return __hiloint2double((int)hi, (int)(mag << 29));
}

template <int V>
__global__ void k(const float *in, double *out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = in[(threadIdx.x + i) & 255];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (V == 0) acc[i] += (double)a[i];
      else if (V == 1) acc[i] += f2d_bits(a[i]);
      else acc[i] *= 1.0000001;
      a[i] = a[i] * 1.0001f + 1e-7f;
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  float *in;
  double *out;
  cudaMalloc(&in, 1024);
  cudaMemset(in, 0, 1024);
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  const char *names[3] = {"F2F.F64.F32 + DADD", "bit-trick f2d + DADD", "DMUL"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (v == 0) k<0><<<148, 384>>>(in, out, iters);
      if (v == 1) k<1><<<148, 384>>>(in, out, iters);
      if (v == 2) k<2><<<148, 384>>>(in, out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 148.0 * 384 * iters * 8;
    printf("%-24s %.3f ms  %.1f Gop/s  %.2f op/clk/SM @1.965GHz\n", names[v], ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
