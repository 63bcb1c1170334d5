// Microbenchmark: the dense operator's A-operand handoff in isolation (no TMA, no epilogue).
// Four "A warps" (one per TMEM lane quarter) write a 128 × 64-column A stage (tf32 hi | lo) to tensor
// memory per chunk with tcgen05.st, then tcgen05.wait::st, tcgen05.fence::before_thread_sync and an
// mbarrier arrive (afull); the MMA thread waits afull, issues tcgen05.fence::after_thread_sync and
// the chunk's 12 MMAs (N = 128, A from that stage) and commits to aempty, which the A warps wait for
// before rewriting the stage — k_cg_persistent.cu's A pipeline.  Modes:
//   0  MMAs only (the A stages never rewritten; no handoff)
//   1  the full handoff (SA stages)
//   2  as 1 without the MMA thread's fence::after_thread_sync
//   3  as 1 with the A warps storing to a scratch region instead of the stage the MMAs read
//      (the same handoff, no write→read dependency)
//   4  as 1 without tcgen05.st (the handoff barriers only)
// Cycles per chunk from clock64 on the MMA thread; SA ∈ {2, 3, 4}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_00420_b200/csrc -o tools/a_handoff_test tools/a_handoff_test.cu
#include <cstdio>
#include "umma.cuh"

using namespace cmtcs::umma;

constexpr int NB = 128;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void arrive(uint64_t *mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}

__global__ void __launch_bounds__(192, 1) k(int mode, int SA, int chunks, unsigned long long *out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t afull[4], aempty[4], done;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  for (int i = t; i < 32768 / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.f;
  if (t == 0) {
    for (int s = 0; s < 4; ++s) { mbar_init(&afull[s], 4); mbar_init(&aempty[s], 1); }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (w == 0) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = slot;
  // TMEM: cross acc [0,128), main acc [128,256), A stages at 256 + 64·s (s < 4)
  if (w == 0) {
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(128, NB);
      const uint64_t bh = desc_sw128(smem_u32(sm)), bl = desc_sw128(smem_u32(sm + 16384));
      const long long c0 = clock64();
      int sa = 0;
      uint32_t ph = 0;
      for (int c = 0; c < chunks; ++c) {
        if (mode != 0) {
          mbar_wait(&afull[sa], ph);
          if (mode != 2) fence_after_sync();
        }
        const uint32_t ta = tm + 256 + 64 * sa;
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          const uint64_t o = (uint64_t)(k8 * 32) >> 4;
          mma_ts(tm, ta + 32 + 8 * k8, bh + o, idesc, 1);
          mma_ts(tm, ta + 8 * k8, bl + o, idesc, 1);
          mma_ts(tm + 128, ta + 8 * k8, bh + o, idesc, 1);
        }
        if (mode != 0) mma_commit(&aempty[sa]);
        if (++sa == SA) { sa = 0; ph ^= 1; }
      }
      mma_commit(&done);
      mbar_wait(&done, 0);
      out[blockIdx.x] = (unsigned long long)(clock64() - c0);
    }
  } else if (w >= 1 && w <= 4 && mode != 0) {
    const int q = (w + 3) & 3;   // warps 1..4 → lane quarters 1, 2, 3, 0 (warp % 4)
    (void)q;
    const uint32_t lane_base = tm + ((uint32_t)((w & 3) * 32) << 16);
    int sa = 0;
    uint32_t ph = 0;
    float v[16];
    for (int i = 0; i < 16; ++i) v[i] = 0.f;
    for (int c = 0; c < chunks; ++c) {
      if (c >= SA) mbar_wait(&aempty[sa], ph ^ 1u);
      fence_after_sync();
      const uint32_t ta = lane_base + (mode == 3 ? 448u : 256u + 64u * (uint32_t)sa);
      if (mode != 4) {
        tmem_st16(ta, v);
        tmem_st16(ta + 16, v);
        tmem_st16(ta + 32, v);
        tmem_st16(ta + 48, v);
        tmem_wait_st();
      }
      fence_before_sync();
      __syncwarp();
      if (lane == 0) arrive(&afull[sa]);
      if (++sa == SA) { sa = 0; ph ^= 1; }
    }
  }
  fence_before_sync();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long *out, h[148];
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  const char *names[5] = {"MMAs only", "handoff (st + fences)", "handoff, no fence::after", "handoff, st elsewhere",
                          "handoff, no st"};
  const int chunks = 2000;
  for (int mode = 0; mode < 5; ++mode)
    for (int SA = 2; SA <= 4; ++SA) {
      if (mode == 0 && SA > 2) continue;
      for (int rep = 0; rep < 2; ++rep) {
        k<<<148, 192, 32768 + 1024>>>(mode, SA, chunks, out);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%-28s SA=%d: %.0f clk per chunk (12 MMAs, N=%d; floor %d)  %s\n", names[mode], SA, (double)mx / chunks, NB,
             12 * NB / 2, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
