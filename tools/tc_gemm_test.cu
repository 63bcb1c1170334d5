// Standalone validation of the tcgen05 3xTF32 GEMM core used by the operator:
//   C[m][n] = Σ_k A[m][k] B[n][k]   (A, B K-major fp32, split into tf32 hi + fp32 lo)
// A tiles by TMA (SWIZZLE_128B), B tiles by TMA or by a cp.async row gather into the same
// swizzled layout, accumulator in TMEM, 3 MMAs (hi·hi + hi·lo + lo·hi) per K=8 step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2310_00420_b200/csrc
//        tools/tc_gemm_test.cu -o tools/tc_gemm_test
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace cmtcs::umma;

constexpr int BM = 128, BKC = 32, ST = 3, THREADS = 128;

template <bool B_TMA, int NACC, bool SEP>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm(const __grid_constant__ CUtensorMap tA_hi, const __grid_constant__ CUtensorMap tA_lo,
           const __grid_constant__ CUtensorMap tB_hi, const __grid_constant__ CUtensorMap tB_lo,
           const float *Bhi, const float *Blo, const int *brow, int K, int N, int NB, float *C, int ldc) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int m0 = blockIdx.x * BM;
  const uint32_t A_BYTES = BM * 128, B_BYTES = NB * 128;
  const uint32_t STAGE = 2 * A_BYTES + 2 * B_BYTES;
  __shared__ uint64_t full[ST], empty[ST];
  __shared__ uint32_t tslot;
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
    prefetch_tmap(&tA_hi); prefetch_tmap(&tA_lo);
    if (B_TMA) { prefetch_tmap(&tB_hi); prefetch_tmap(&tB_lo); }
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tslot;
  const int nk = (K + BKC - 1) / BKC;
  const uint32_t idesc = idesc_tf32(128, N);

  auto issue = [&](int st, int kc) {
    unsigned char *base = sm + st * STAGE;
    const int k0 = kc * BKC;
    if (tid == 0) {
      mbar_arrive_expect_tx(&full[st], 2 * A_BYTES + (B_TMA ? 2 * B_BYTES : 0));
      tma_load_2d(base, &tA_hi, k0, m0, &full[st]);
      tma_load_2d(base + A_BYTES, &tA_lo, k0, m0, &full[st]);
      if (B_TMA) {
        tma_load_2d(base + 2 * A_BYTES, &tB_hi, k0, 0, &full[st]);
        tma_load_2d(base + 2 * A_BYTES + B_BYTES, &tB_lo, k0, 0, &full[st]);
      }
    }
    if (!B_TMA) {
      // gather rows brow[j] of B (hi, lo): NB rows x 8 chunks of 16 B each
      const uint32_t sb = smem_u32(base + 2 * A_BYTES);
      for (int e = tid; e < NB * 8; e += THREADS) {
        const int j = e >> 3, c = e & 7;
        const int k = k0 + 4 * c;
        const bool ok = j < N && k < K;
        const size_t off = ok ? (size_t)brow[j] * K + k : 0;
        cp_async16(sb + sw128_offset(j, c), Bhi + off, ok);
        cp_async16(sb + B_BYTES + sw128_offset(j, c), Blo + off, ok);
      }
    }
  };

  for (int s = 0; s < ST - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    const int st = kc % ST;
    mbar_wait(&full[st], (kc / ST) & 1);
    if (!B_TMA) {
      cp_wait<ST - 2>();
      fence_proxy_async();
    }
    __syncthreads();
    if (tid == 0) {
      fence_after_sync();
      unsigned char *base = sm + st * STAGE;
      const uint64_t ah = desc_sw128(smem_u32(base)), al = desc_sw128(smem_u32(base + A_BYTES));
      const uint64_t bh = desc_sw128(smem_u32(base + 2 * A_BYTES)), bl = desc_sw128(smem_u32(base + 2 * A_BYTES + B_BYTES));
      const int q = (kc * NACC) / nk;                    // K-quarter → its own accumulator
      const int qfirst = (q * nk + NACC - 1) / NACC;      // first chunk of this accumulator
      const uint32_t tm_main = tmem + q * (SEP ? 2 : 1) * 128;
      const uint32_t tm_x = SEP ? tm_main + 128 : tm_main;
#pragma unroll
      for (int k8 = 0; k8 < BKC / 8; ++k8) {
        const uint64_t o = (uint64_t)(k8 * 32) >> 4;  // +32 bytes per K=8 step inside the swizzled row
        const uint32_t first = (kc == qfirst && k8 == 0) ? 0u : 1u;
        mma_tf32(tm_x, al + o, bh + o, idesc, first);
        mma_tf32(tm_x, ah + o, bl + o, idesc, 1u);
        mma_tf32(tm_main, ah + o, bh + o, idesc, SEP ? first : 1u);
      }
      mma_commit(&empty[st]);
    }
    const int nx = kc + ST - 1;
    if (nx < nk) {
      const int ns = nx % ST;
      if (nx >= ST) mbar_wait(&empty[ns], ((nx - ST) / ST) & 1);
      issue(ns, nx);
    }
    cp_commit();
  }
  mbar_wait(&empty[(nk - 1) % ST], ((nk - 1) / ST) & 1);
  fence_after_sync();
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows), 16 columns at a time
  const int row = m0 + warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 16) {
    float tot[16];
    for (int i = 0; i < 16; ++i) tot[i] = 0.f;
    // sum the small accumulators first, the main ones last
    for (int pass = SEP ? 1 : 0; pass >= 0; --pass)
      for (int q = 0; q < NACC; ++q) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + q * (SEP ? 2 : 1) * 128 + pass * 128 + c0, v);
        for (int i = 0; i < 16; ++i) tot[i] += v[i];
      }
    for (int i = 0; i < 16; ++i)
      if (c0 + i < N) C[(size_t)row * ldc + c0 + i] = tot[i];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

__global__ void k_split(const float *x, float *hi, float *lo, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float h = tf32_hi(x[i]);
    hi[i] = h;
    lo[i] = x[i] - h;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return (EncodeFn)fn;
}

static CUtensorMap make_map(EncodeFn enc, const float *p, int K, int rows, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)p, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}

template <int NACC, bool SEP>
int run(int M, int N, int NB, int K, bool btma) {
  std::vector<float> A((size_t)M * K), B((size_t)NB * K);
  srand(1234);
  for (auto &x : A) x = (float)rand() / RAND_MAX * 2.f - 1.f;
  for (auto &x : B) x = (float)rand() / RAND_MAX * 2.f - 1.f;
  std::vector<int> rows(NB);
  for (int j = 0; j < NB; ++j) rows[j] = btma ? j : (NB - 1 - j);  // gather reverses the rows
  float *dA, *dB, *Ah, *Al, *Bh, *Bl, *dC;
  int *drow;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&Ah, A.size() * 4); cudaMalloc(&Al, A.size() * 4);
  cudaMalloc(&Bh, B.size() * 4); cudaMalloc(&Bl, B.size() * 4);
  cudaMalloc(&dC, (size_t)M * N * 4); cudaMalloc(&drow, NB * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(drow, rows.data(), NB * 4, cudaMemcpyHostToDevice);
  k_split<<<256, 256>>>(dA, Ah, Al, A.size());
  k_split<<<256, 256>>>(dB, Bh, Bl, B.size());
  EncodeFn enc = get_encode();
  CUtensorMap tAh = make_map(enc, Ah, K, M, 128), tAl = make_map(enc, Al, K, M, 128);
  CUtensorMap tBh = make_map(enc, Bh, K, NB, NB), tBl = make_map(enc, Bl, K, NB, NB);
  const size_t smem = 1024 + (size_t)ST * (2 * 128 * 128 + 2 * NB * 128);
  auto kern = btma ? k_gemm<true, NACC, SEP> : k_gemm<false, NACC, SEP>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<M / 128, THREADS, smem>>>(tAh, tAl, tBh, tBl, Bh, Bl, drow, K, N, NB, dC, N);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> Cg((size_t)M * N);
  cudaMemcpy(Cg.data(), dC, Cg.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0, maxerr32 = 0;
  for (int m = 0; m < M; ++m) {
    if (M > 1024 && m >= 256 && m < M - 128) continue;  // sample rows of the big case
    for (int n = 0; n < N; ++n) {
      double s = 0;
      float s32 = 0;
      const int br = rows[n];
      for (int k = 0; k < K; ++k) {
        s += (double)A[(size_t)m * K + k] * B[(size_t)br * K + k];
        s32 = fmaf(A[(size_t)m * K + k], B[(size_t)br * K + k], s32);
      }
      maxerr = fmax(maxerr, fabs(Cg[(size_t)m * N + n] - s));
      maxerr32 = fmax(maxerr32, fabs((double)s32 - s));
      maxref = fmax(maxref, fabs(s));
    }
  }
  printf("{\"nacc\": %d, \"sep\": %d, \"M\": %d, \"N\": %d, \"K\": %d, \"b_tma\": %d, \"err\": \"%s\", \"rel_err_3xtf32\": %.3e, \"rel_err_fp32_serial\": %.3e}\n",
         NACC, (int)SEP, M, N, K, (int)btma, cudaGetErrorString(e), maxerr / maxref, maxerr32 / maxref);
  // timing
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) kern<<<M / 128, THREADS, smem>>>(tAh, tAl, tBh, tBl, Bh, Bl, drow, K, N, NB, dC, N);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"time_us\": %.2f, \"eff_tflops\": %.2f}\n", ms * 100, 2.0 * M * N * K / (ms / 10 * 1e-3) / 1e12);
  cudaFree(dA); cudaFree(dB); cudaFree(Ah); cudaFree(Al); cudaFree(Bh); cudaFree(Bl); cudaFree(dC); cudaFree(drow);
  return e == cudaSuccess ? 0 : 1;
}

int main() {
  int rc = 0;
  rc |= run<1, false>(256, 96, 96, 1024, true);
  rc |= run<1, false>(256, 80, 96, 1024, false);
  rc |= run<1, false>(148 * 128, 96, 96, 4096, true);
  rc |= run<1, true>(148 * 128, 96, 96, 4096, true);
  rc |= run<2, false>(148 * 128, 96, 96, 4096, true);
  rc |= run<2, true>(148 * 128, 96, 96, 4096, true);
  rc |= run<1, true>(256, 96, 96, 1024, true);
  rc |= run<2, true>(1024, 96, 96, 256, true);
  return rc;
}
