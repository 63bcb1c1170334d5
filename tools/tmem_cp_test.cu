// Microbenchmark + check: staging the A operand (128 × 32 fp32 K-major SW128 tile) into tensor memory
// by tcgen05.cp (smem → TMEM on the tensor pipe, issued by the MMA thread in order with its MMAs)
// instead of tcgen05.st from registers (the A warps' path in k_cg_persistent.cu).
//   part 1: correctness — D = A·Bᵀ (M = N = 128, K = 32) with A in TMEM written (a) by tcgen05.st
//           row per thread, (b) by 4 × tcgen05.cp.128x256b from the SW128 tile; max |D_a − D_b| and
//           |D − D_ref| (host fp64 reference; tf32-exact inputs)
//   part 2: throughput of the operator's per-chunk MMA sequence (12 MMAs, N = 128) with A staged
//           every chunk: mode 0 MMAs only; mode 1 + 4 warps streaming tcgen05.st (32 KB per chunk
//           pace-free); mode 2 + the MMA thread issuing 8 tcgen05.cp (32 KB) per chunk before its MMAs
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2310_00420_b200/csrc -o tools/tmem_cp_test tools/tmem_cp_test.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "umma.cuh"

using namespace cmtcs::umma;

constexpr int NB = 128;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_cp(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void st16(uint32_t taddr, float x) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr), "f"(x)
      : "memory");
}

// part 1: A (SW128 tile at sm), B (SW128 tile at sm + 16 KB); out[0..128*128) D via st, [..2*) D via cp
__global__ void __launch_bounds__(128, 1) k_check(const float *A, const float *B, float *out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, w = t >> 5;
  // swizzled K-major tiles: element (r, k) at sw128_offset(r, k/4) + (k%4)*4
  for (int i = t; i < 128 * 32; i += 128) {
    const int r = i / 32, kk = i % 32;
    *reinterpret_cast<float *>(sm + sw128_offset(r, kk / 4) + (kk % 4) * 4) = A[i];
    *reinterpret_cast<float *>(sm + 16384 + sw128_offset(r, kk / 4) + (kk % 4) * 4) = B[i];
  }
  if (t == 0) mbar_init(&done, 1);
  if (w == 0) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = slot, ta_st = tm + 256, ta_cp = tm + 320;
  // (a) tcgen05.st: thread t writes row t
  {
    float v[16];
    for (int h = 0; h < 2; ++h) {
      for (int i = 0; i < 16; ++i) v[i] = A[t * 32 + 16 * h + i];
      tmem_st16(ta_st + ((uint32_t)(w * 32) << 16) + 16 * h, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (t == 0) {
    const uint64_t ad = desc_sw128(smem_u32(sm)), bd = desc_sw128(smem_u32(sm + 16384));
    for (int k8 = 0; k8 < 4; ++k8) tmem_cp(ta_cp + 8 * k8, ad + ((uint64_t)(k8 * 32) >> 4));   // (b)
    const uint32_t idesc = idesc_tf32(128, NB);
    for (int k8 = 0; k8 < 4; ++k8) {
      const uint64_t o = (uint64_t)(k8 * 32) >> 4;
      mma_ts(tm, ta_st + 8 * k8, bd + o, idesc, k8 ? 1u : 0u);
      mma_ts(tm + 128, ta_cp + 8 * k8, bd + o, idesc, k8 ? 1u : 0u);
    }
    mma_commit(&done);
  }
  mbar_wait(&done, 0);
  fence_after_sync();
  for (int c0 = 0; c0 < 256; c0 += 16) {
    float v[16];
    tmem_ld16(tm + ((uint32_t)(w * 32) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) out[(c0 / 128) * 16384 + t * 128 + (c0 % 128) + i] = v[i];
  }
  fence_before_sync();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tm);
}

__global__ void __launch_bounds__(384, 1) k_rate(int mode, int chunks, unsigned long long *out) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 98304 / 4; i += blockDim.x) reinterpret_cast<float *>(sm)[i] = 0.f;
  if (t == 0) { mbar_init(&done, 1); stop = 0; }
  if (w == 0) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = slot;
  if (t == 0 && mode == 5) {   // store stream alone: thread 0 just waits ~chunks*768 cycles
    const long long c0 = clock64();
    while (clock64() - c0 < (long long)chunks * 768) {}
    out[blockIdx.x] = (unsigned long long)(clock64() - c0);
    stop = 1;
  } else if (t == 0) {
    const uint32_t idesc = idesc_tf32(128, NB);
    // B hi | lo at sm + 32 KB (2 × 16 KB), A hi | lo tiles at sm (2 × 16 KB) for the copies
    const uint64_t bh = desc_sw128(smem_u32(sm + 32768)), bl = desc_sw128(smem_u32(sm + 49152));
    const uint64_t ah = desc_sw128(smem_u32(sm)), al = desc_sw128(smem_u32(sm + 16384));
    const uint32_t tx = tm, tmain = tm + 128;
    const long long c0 = clock64();
    for (int c = 0; c < chunks; ++c) {
      const uint32_t ta = tm + 384 + 64 * (c & 1);
      if (mode == 2) {
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          tmem_cp(ta + 8 * k8, ah + ((uint64_t)(k8 * 32) >> 4));
          tmem_cp(ta + 32 + 8 * k8, al + ((uint64_t)(k8 * 32) >> 4));
        }
      }
#pragma unroll
      for (int k8 = 0; k8 < 4; ++k8) {
        const uint64_t o = (uint64_t)(k8 * 32) >> 4;
        mma_ts(tx, ta + 32 + 8 * k8, bh + o, idesc, 1);
        mma_ts(tx, ta + 8 * k8, bl + o, idesc, 1);
        mma_ts(tmain, ta + 8 * k8, bh + o, idesc, 1);
      }
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    const long long c1 = clock64();
    out[blockIdx.x] = (unsigned long long)(c1 - c0);
    stop = 1;
  } else if (w >= 8 && (mode == 1 || mode >= 3)) {
    // (mode 5: the stream of mode 3 with no MMAs running)
    // mode 1: stores to columns 256..319 (away from the A operand); mode 3: to the OTHER A stage
    // (384 + 64·((c+1)&1) — what the kernel's A warps do); mode 4: into the A stage being read
    const uint32_t col = mode == 1 ? 256u : 384u;   // modes 3, 4, 5: the A stages
    const uint32_t lane_base = tm + ((uint32_t)((w & 3) * 32) << 16) + col;
    float x = 0.f;
    int it = 0;
    const long long s0 = clock64();
    while (!stop) {
      const uint32_t off = mode == 1 ? 0u : (mode == 3 ? 64u * (uint32_t)((it + 1) & 1) : 64u * (uint32_t)(it & 1));
      st16(lane_base + off, x);
      st16(lane_base + off + 16, x);
      st16(lane_base + off + 32, x);
      st16(lane_base + off + 48, x);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      x += 1.f;
      ++it;
    }
    const long long s1 = clock64();
    if ((threadIdx.x & 31) == 0 && w == 8) out[148 + blockIdx.x] = (unsigned long long)((s1 - s0) / (it > 0 ? it : 1));
  }
  fence_before_sync();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tm);
}

int main() {
  // part 1
  const int n = 128 * 32;
  float *hA = (float *)malloc(n * 4), *hB = (float *)malloc(n * 4), *hD = (float *)malloc(2 * 16384 * 4);
  srand(7);
  for (int i = 0; i < n; ++i) {
    hA[i] = (float)((rand() % 2001) - 1000) / 256.f;   // tf32-exact small integers / 256
    hB[i] = (float)((rand() % 2001) - 1000) / 512.f;
  }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, n * 4); cudaMalloc(&dB, n * 4); cudaMalloc(&dD, 2 * 16384 * 4);
  cudaMemcpy(dA, hA, n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, n * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  k_check<<<1, 128, 32768 + 1024>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, dD, 2 * 16384 * 4, cudaMemcpyDeviceToHost);
  double e_st = 0, e_cp = 0, e_ab = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 128; ++c) {
      double ref = 0;
      for (int k = 0; k < 32; ++k) ref += (double)hA[r * 32 + k] * hB[c * 32 + k];
      e_st = fmax(e_st, fabs(hD[r * 128 + c] - ref));
      e_cp = fmax(e_cp, fabs(hD[16384 + r * 128 + c] - ref));
      e_ab = fmax(e_ab, fabs(hD[r * 128 + c] - hD[16384 + r * 128 + c]));
    }
  printf("check (%s): max |D_st - ref| %.3g, |D_cp - ref| %.3g, |D_st - D_cp| %.3g\n", cudaGetErrorString(e), e_st,
         e_cp, e_ab);
  // part 2
  unsigned long long *out, h[296];
  cudaMalloc(&out, 296 * 8);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  const char *names[6] = {"MMAs only", "+ tcgen05.st stream (4 warps)", "+ 8 tcgen05.cp per chunk",
                          "+ st stream into the other A stage", "+ st stream over both A stages", "st stream alone"};
  const int chunks = 2000;
  for (int mode = 0; mode < 6; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(out + 148, 0, 148 * 8);
      k_rate<<<148, 384, 98304 + 1024>>>(mode, chunks, out);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    unsigned long long smx = 0;
    for (int i = 148; i < 296; ++i) smx = h[i] > smx ? h[i] : smx;
    printf("%-36s: %.0f clk per chunk (12 MMAs, N=%d; floor %d); store warp: %llu clk per 32 KB-per-CTA round  %s\n",
           names[mode], (double)mx / chunks, NB, 12 * NB / 2, smx, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
