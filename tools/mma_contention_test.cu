// Microbenchmark: the CG operator's per-chunk MMA sequence (3xTF32: per K = 8 step lo·hi and hi·lo
// into the cross accumulator, hi·hi into the main one; A in TMEM, B hi/lo in shared memory, N = 80)
// issued by one thread, alone and with concurrent TMEM traffic from other warps:
//   mode 0: MMAs only
//   mode 1: + 4 warps streaming tcgen05.ld of another TMEM region (an epilogue draining)
//   mode 2: + 4 warps streaming tcgen05.st into another TMEM region (A warps writing A stages)
//   mode 3: + both (8 warps)
//   mode 4: + 4 warps streaming ld.shared (shared-memory port pressure)
//   mode 5: + 4 warps streaming DMMA (the fp64 mean columns' FP64 tensor path)
//   mode 6: + 4 warps streaming F2F.F64.F32 + DMMA
//   mode 7: MMAs + a tcgen05.commit to an mbarrier after every chunk (not waited)
//   mode 8: MMAs + commit after every chunk, waiting for it before the next chunk (issue → done)
//   mode 9: as mode 0, but the whole warp runs the issue loop and one elected lane issues each MMA
//           (warp-uniform operands: no per-MMA register → uniform-register moves)
//   mode 10: as mode 9 with the main accumulator at TMEM column 80 (16- but not 32-aligned)
//   mode 11: as mode 9 plus the kernel's per-chunk overhead: two completed-mbarrier waits,
//            tcgen05.fence::after_thread_sync, two integer divisions, two commits
// Cycles per chunk (12 MMAs) from clock64 on the issuing thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_00420_b200/csrc -o tools/mma_contention_test tools/mma_contention_test.cu
#include <cstdio>
#include "umma.cuh"

using namespace cmtcs::umma;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void st16(uint32_t taddr, float x) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr), "f"(x)
      : "memory");
}

constexpr int NB = 80;

__global__ void __launch_bounds__(384, 1) k(int mode, int chunks, unsigned long long *out, float *sink) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t done, cdone;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.f;
  if (t == 0) { mbar_init(&done, 1); mbar_init(&cdone, 1); stop = 0; }
  if (w == 0) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = slot;
  if (mode == 11 && w == 0) {
    const uint32_t idesc = idesc_tf32(128, NB);
    const uint64_t bh = desc_sw128(smem_u32(sm)), bl = desc_sw128(smem_u32(sm + NB * 128));
    const uint32_t tx = tm, tmain = tm + 96, ta = tm + 384;
    __shared__ uint64_t pre;
    if (t == 0) { mbar_init(&pre, 1); asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&pre)) : "memory"); }
    __syncwarp();
    const long long c0 = clock64();
    int nk = chunks, nacc = 1;
    for (int c = 0; c < chunks; ++c) {
      mbar_wait(&pre, 0);
      mbar_wait(&pre, 0);
      fence_after_sync();
      const int q = (c * nacc) / nk;
      const int qfirst = (q * nk + nacc - 1) / nacc;
#pragma unroll
      for (int k8 = 0; k8 < 4; ++k8) {
        const uint64_t o = (uint64_t)(k8 * 32) >> 4;
        mma_ts_elect(tx, ta + 32 + 8 * k8, bh + o, idesc, 1);
        mma_ts_elect(tx, ta + 8 * k8, bl + o, idesc, 1);
        mma_ts_elect(tmain + 0 * q, ta + 8 * k8, bh + o, idesc, (c == qfirst && k8 == 0) ? 0u : 1u);
      }
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&done)) : "memory");
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&done)) : "memory");
      __syncwarp();
    }
    const long long c1 = clock64();
    if (t == 0) { out[blockIdx.x] = (unsigned long long)(c1 - c0); stop = 1; }
  } else if ((mode == 9 || mode == 10) && w == 0) {
    const uint32_t idesc = idesc_tf32(128, NB);
    const uint64_t bh = desc_sw128(smem_u32(sm)), bl = desc_sw128(smem_u32(sm + NB * 128));
    const uint32_t tx = tm, tmain = tm + (mode == 10 ? 80 : 96), ta = tm + 384;
    const long long c0 = clock64();
    for (int c = 0; c < chunks; ++c) {
#pragma unroll
      for (int k8 = 0; k8 < 4; ++k8) {
        const uint64_t o = (uint64_t)(k8 * 32) >> 4;
        mma_ts_elect(tx, ta + 32 + 8 * k8, bh + o, idesc, 1);
        mma_ts_elect(tx, ta + 8 * k8, bl + o, idesc, 1);
        mma_ts_elect(tmain, ta + 8 * k8, bh + o, idesc, 1);
      }
    }
    if (t == 0) mma_commit(&done);
    mbar_wait(&done, 0);
    const long long c1 = clock64();
    if (t == 0) { out[blockIdx.x] = (unsigned long long)(c1 - c0); stop = 1; }
  } else if (t == 0 && mode < 9) {
    const uint32_t idesc = idesc_tf32(128, NB);
    const uint64_t bh = desc_sw128(smem_u32(sm)), bl = desc_sw128(smem_u32(sm + NB * 128));
    const uint32_t tx = tm, tmain = tm + 96, ta = tm + 384;
    const long long c0 = clock64();
    for (int c = 0; c < chunks; ++c) {
#pragma unroll
      for (int k8 = 0; k8 < 4; ++k8) {
        const uint64_t o = (uint64_t)(k8 * 32) >> 4;
        mma_ts(tx, ta + 32 + 8 * k8, bh + o, idesc, 1);
        mma_ts(tx, ta + 8 * k8, bl + o, idesc, 1);
        mma_ts(tmain, ta + 8 * k8, bh + o, idesc, 1);
      }
      if (mode == 7 || mode == 8) mma_commit(&cdone);
      if (mode == 8) mbar_wait(&cdone, c & 1);
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    const long long c1 = clock64();
    out[blockIdx.x] = (unsigned long long)(c1 - c0);
    stop = 1;
  } else if (w >= 4 && w < 8 && (mode == 1 || mode == 3)) {
    float acc = 0.f;
    const uint32_t lane_base = tm + ((uint32_t)((w & 3) * 32) << 16) + 192;
    while (!stop) {
      float v[16];
      tmem_ld16(lane_base + (acc > 1e30f ? 16 : 0), v);
      for (int i = 0; i < 16; ++i) acc += v[i];
    }
    if (acc == 1.2345f) sink[0] = acc;
  } else if (w >= 8 && (mode == 2 || mode == 3)) {
    const uint32_t lane_base = tm + ((uint32_t)((w & 3) * 32) << 16) + 448;
    float x = 0.f;
    while (!stop) {
      st16(lane_base, x);
      st16(lane_base + 16, x);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      x += 1.f;
    }
  } else if (w >= 4 && w < 8 && (mode == 5 || mode == 6)) {
    double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    float fa = (float)(t & 7);
    double b = 1.0;
    while (!stop) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double a = mode == 6 ? (double)(fa + (float)i) : 1.0 + i;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
      }
      fa += 1.f;
    }
    if (acc[0][0] == 1.2345) sink[0] = (float)acc[1][1];
  } else if (w >= 4 && w < 8 && mode == 4) {
    float acc = 0.f;
    uint32_t a = smem_u32(sm) + 32768 + (t & 127) * 16;
    while (!stop) {
      float4 v;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
      acc += v.x;
      a ^= 2048;
    }
    if (acc == 1.2345f) sink[0] = acc;
  }
  fence_before_sync();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long *out, h[148];
  float *sink;
  cudaMalloc(&out, 148 * 8);
  cudaMalloc(&sink, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const char *names[12] = {"MMAs only", "+ tcgen05.ld stream", "+ tcgen05.st stream", "+ ld and st streams", "+ ld.shared stream",
                          "+ DMMA stream", "+ F2F + DMMA stream", "commit per chunk", "commit + wait per chunk",
                          "whole warp, elect.sync", "elect, main acc at col 80", "elect + kernel overheads"};
  const int chunks = 2000;
  for (int mode = 0; mode < 12; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      k<<<148, 384, 65536 + 1024>>>(mode, chunks, out, sink);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-22s: %.0f clk per chunk (12 MMAs, N=%d; floor 12*%d = %d)  %s\n", names[mode], (double)mx / chunks, NB, NB / 2,
           12 * NB / 2, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
