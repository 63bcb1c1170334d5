// Microbenchmark: tcgen05.mma kind::tf32 issue-to-completion throughput for M = 128 and several N,
// A from TMEM (TS) vs A from shared memory (SS), B from shared memory.  148 CTAs, one thread issues
// `reps` MMAs (K = 8 each) into one accumulator, one commit; cycles per MMA from clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_00420_b200/csrc -o tools/mma_rate_test tools/mma_rate_test.cu
#include <cstdio>
#include "umma.cuh"

using namespace cmtcs::umma;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}

template <int ND, int TS>
__global__ void k(int N, int reps, unsigned long long *out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const int t = threadIdx.x;
  for (int i = t; i < (16384 + 256 * 128) / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.f;
  if (t == 0) mbar_init(&done, 1);
  if (t < 32) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = slot;
  if (t == 0) {
    const uint32_t idesc = idesc_tf32(128, N);
    const uint64_t ad = desc_sw128(smem_u32(sm)), bd = desc_sw128(smem_u32(sm + 16384));
    const long long c0 = clock64();
    for (int i = 0; i < reps; i += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t o = (uint64_t)(j * 32) >> 4;
        const uint32_t dcol = (uint32_t)((j % ND) * (ND > 1 ? 384 / ND / 16 * 16 : 0));
        if (TS) mma_ts(tm + dcol, tm + 384 + 8 * j, bd + o, idesc, 1);
        else mma_tf32(tm + dcol, ad + o, bd + o, idesc, 1);
      }
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    const long long c1 = clock64();
    out[blockIdx.x] = (unsigned long long)(c1 - c0);
  }
  fence_before_sync();
  __syncthreads();
  if (t < 32) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long *out, h[148];
  cudaMalloc(&out, 148 * 8);
  typedef void (*K)(int, int, unsigned long long *);
  K ks[2][3] = {{k<1, 0>, k<2, 0>, k<4, 0>}, {k<1, 1>, k<2, 1>, k<4, 1>}};
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) cudaFuncSetAttribute(ks[a][b], cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 256 * 128 + 1024);
  const int Ns[] = {80, 128, 160, 256};
  const int reps = 4096;
  for (int ts = 0; ts < 2; ++ts)
   for (int nd = 1; nd <= 4; nd *= 2)
    for (int N : Ns) {
      if (N * nd > 384 && nd > 1) continue;
      for (int rep = 0; rep < 2; ++rep) {
        ks[ts][nd == 1 ? 0 : nd == 2 ? 1 : 2]<<<148, 128, 16384 + 256 * 128 + 1024>>>(N, reps, out);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%s %d accumulators N=%3d: %.1f clk per MMA (floor 128*N/256 = %d)  %s\n", ts ? "TS (A in TMEM)" : "SS (A in smem)", nd, N,
             (double)mx / reps, N / 2, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
