// Microbenchmark: per-chunk cost of an empty mbarrier ring (producer lane → 2 converter warps →
// issuer lane → producer), the synchronisation skeleton of k_cg_persistent's K loop, on 148 CTAs
// of 384 threads.  Variants: ring depth S, the issuer "arrive" vs a tcgen05.commit-free arrive,
// idle warps parked at a barrier vs spinning.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ring_test tools/ring_test.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t *m, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(m)), "r"(c) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(m)) : "memory");
}
template <int V>
__device__ __forceinline__ void wait(uint64_t *m, uint32_t ph) {
  const uint32_t a = su32(m);
  if (V == 0) {
    asm volatile("{\n\t.reg .pred done;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t@!done bra W_%=;\n\t}\n" ::"r"(a), "r"(ph) : "memory");
  } else if (V == 1) {
    asm volatile("{\n\t.reg .pred done;\nW_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 done, [%0], %1;\n\t@!done bra W_%=;\n\t}\n" ::"r"(a), "r"(ph) : "memory");
  } else {
    asm volatile("{\n\t.reg .pred done;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, %2;\n\t@!done bra W_%=;\n\t}\n" ::"r"(a), "r"(ph), "r"(1000) : "memory");
  }
}

template <int V>
__global__ void __launch_bounds__(384, 1) k(int nchunks, int S, unsigned long long *out) {
  __shared__ uint64_t full[8], conv[8], empty[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { init(&full[s], 1); init(&conv[s], 2); init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (warp == 0 && lane == 0) {
    int st = 0; uint32_t ph = 0;
    for (int g = 0; g < nchunks; ++g) {
      if (g >= S) wait<V>(&empty[st], ph ^ 1u);
      arrive(&full[st]);
      if (++st == S) { st = 0; ph ^= 1u; }
    }
  } else if (warp == 1 && lane == 0) {
    int st = 0; uint32_t ph = 0;
    for (int g = 0; g < nchunks; ++g) {
      wait<V>(&conv[st], ph);
      arrive(&empty[st]);
      if (++st == S) { st = 0; ph ^= 1u; }
    }
  } else if (warp == 2 || warp == 3) {
    int st = 0; uint32_t ph = 0;
    for (int g = 0; g < nchunks; ++g) {
      wait<V>(&full[st], ph);
      __syncwarp();
      if (lane == 0) arrive(&conv[st]);
      if (++st == S) { st = 0; ph ^= 1u; }
    }
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[blockIdx.x] = t1 - t0;
  }
}

int main() {
  unsigned long long *out, h[148];
  cudaMalloc(&out, 148 * 8);
  const int n = 20000;
  for (int v = 0; v < 3; ++v)
    for (int S = 2; S <= 4; ++S) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) k<0><<<148, 384>>>(n, S, out);
        if (v == 1) k<1><<<148, 384>>>(n, S, out);
        if (v == 2) k<2><<<148, 384>>>(n, S, out);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("wait=%s S=%d: %.1f ns per chunk (%s)\n", v == 0 ? "try_wait" : v == 1 ? "test_wait" : "try_wait+hint", S,
             (double)mx / n, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
