// Microbenchmark of the ALU roofline denominators on this GPU: FP32 FFMA, packed FFMA2
// (fma.rn.f32x2, sm_100+) and FP64 DFMA throughput, all SMs, CUDA-event timed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fma_peak.cu -o tools/fma_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int ACC = 8;

__global__ void k_ffma(float *out, float a, float b) {
  float acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float x = a + threadIdx.x * 1e-7f, y = b;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = fmaf(acc[i], x, y);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += acc[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void k_ffma2(float *out, float a, float b) {
  unsigned long long acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) {
    float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    acc[i] = *reinterpret_cast<unsigned long long *>(&v);
  }
  float2 xv = make_float2(a + threadIdx.x * 1e-7f, a), yv = make_float2(b, b);
  unsigned long long x = *reinterpret_cast<unsigned long long *>(&xv), y = *reinterpret_cast<unsigned long long *>(&yv);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = ffma2(acc[i], x, y);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) {
    float2 v = *reinterpret_cast<float2 *>(&acc[i]);
    s += v.x + v.y;
  }
  if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void k_dfma(float *out, double a, double b) {
  double acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  double x = a + threadIdx.x * 1e-9, y = b;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = fma(acc[i], x, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += acc[i];
  if (s == 12345.0) out[threadIdx.x] = (float)s;
}

template <class F>
double run(F launch, double flop_per_thread, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) launch();
  cudaEventRecord(e0);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return flop_per_thread * blocks * threads * reps / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out;
  cudaMalloc(&out, 4096);
  const int threads = 256, blocks = sms * 8;
  double f32 = run([&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 2.0 * ITERS * ACC, blocks, threads);
  double f32x2 = run([&] { k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 4.0 * ITERS * ACC, blocks, threads);
  double f64 = run([&] { k_dfma<<<blocks, threads>>>(out, 0.999, 1e-3); }, 2.0 * ITERS * ACC, blocks, threads);
  cudaError_t e = cudaDeviceSynchronize();
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"dfma_tflops\": %.2f, \"err\": \"%s\"}\n",
         sms, clk, f32, f32x2, f64, cudaGetErrorString(e));
  return 0;
}
