// Microbenchmark: cost of one grid-wide barrier over 148 co-resident CTAs (128 threads each) on
// the B200, for the barrier variants considered for the persistent CG kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridbar_test tools/gridbar_test.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

template <int V>
__device__ __forceinline__ void bar_sync(unsigned *bar, unsigned &epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    epoch += 1;
    const unsigned target = epoch * gridDim.x;
    if (V == 0) __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    if (V == 0) __threadfence();
  }
  __syncthreads();
}

template <int V>
__global__ void k_bar(unsigned *bar, int iters, unsigned long long *out) {
  unsigned epoch = 0;
  unsigned long long t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (V == 2) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
  } else {
    for (int i = 0; i < iters; ++i) bar_sync<V>(bar, epoch);
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

template <int V>
void run(const char *name, int grid, unsigned *bar, unsigned long long *out) {
  const int iters = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(bar, 0, 4);
    void *args[] = {&bar, (void *)&iters, &out};
    cudaLaunchCooperativeKernel((void *)k_bar<V>, grid, 128, args, 0, 0);
    cudaDeviceSynchronize();
  }
  unsigned long long ns;
  cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
  printf("%-40s grid %d: %.3f us per barrier (%s)\n", name, grid, ns * 1e-3 / iters,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned *bar;
  unsigned long long *out;
  cudaMalloc(&bar, 4);
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("red.release/ld.acquire + threadfence", sms, bar, out);
  run<1>("red.release/ld.acquire", sms, bar, out);
  run<2>("cooperative_groups grid.sync", sms, bar, out);
  run<1>("red.release/ld.acquire", 64, bar, out);
  return 0;
}
