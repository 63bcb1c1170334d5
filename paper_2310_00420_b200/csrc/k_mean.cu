// Φμ for ℓ (Eq. 3 via reading A1): Um[t][n][c] = Σ_d Φ_t[n][d] · μ_tc[d] in fp64 for the final means
// of an E-step (inside the CG loop the mean columns are computed on the CUDA cores of the persistent
// CG kernel, k_cg_persistent.cu).  DFMA on fp32 Φ tiles streamed through a 3-stage cp.async ring;
// split-K over S1 slices, the S1 CTAs of a row tile form a cluster and reduce over DSMEM.
#include <cooperative_groups.h>

#include "cmtcs_internal.cuh"

namespace cg = cooperative_groups;

namespace cmtcs {

namespace {

constexpr int BR = OP_BR;       // 128 rows per CTA
constexpr int BK = OP_BK;       // 16: contraction chunk
constexpr int ST = 3;           // pipeline stages
constexpr int A1LD = BK + 4;    // stage-1 A tile [r][k]

struct __align__(16) SmemM1 {
  float A[ST][BR][A1LD];
  double Bm[ST][BK][MAXC];
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;  // src-size 0 ⇒ zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// stage 1:  grid (1, nRT1 * S1, Tl), clusters of (1, S1, 1)
__global__ void __launch_bounds__(OP_THREADS) k_mu_stage1(KParams p, const double *__restrict__ mu_src) {
  extern __shared__ __align__(16) unsigned char dsm1[];
  SmemM1 &sm = *reinterpret_cast<SmemM1 *>(dsm1);
  const Dims &d = p.d;
  const int t = blockIdx.z, tid = threadIdx.x;
  const int rt = blockIdx.y / d.S1, sp = blockIdx.y % d.S1;
  const int N = d.N, D = d.D, C = d.C;
  const float *__restrict__ phi = p.phi + (size_t)t * d.phi_task_stride;
  const int n0 = rt * BR;
  const int kb = sp * d.K1, ke = min(D, kb + d.K1);
  const int nk = (ke - kb + BK - 1) / BK;

  // A tile: Φ[n0 + r][k0 .. k0+15] → A[r][0..15]  (2 × 16-byte cp.async per thread)
  auto loadA = [&](int buf, int k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * OP_THREADS, r = idx >> 2, q = idx & 3;
      const int n = n0 + r, k = k0 + 4 * q;
      const bool ok = n < N && k < ke;
      cp_async16(&sm.A[buf][r][4 * q], ok ? phi + (size_t)n * D + k : phi, ok);
    }
  };
  const double *src = mu_src + (size_t)t * C * D;
  const int r = tid & (BR - 1), h = tid >> 7;
  double acc[MAXC / 2];
#pragma unroll
  for (int i = 0; i < MAXC / 2; ++i) acc[i] = 0.0;
  auto loadB = [&](int buf, int k0) {
    if (tid < BK * C) {
      const int c = tid / BK, kk = tid % BK;
      sm.Bm[buf][kk][c] = (k0 + kk < ke) ? src[(size_t)c * D + k0 + kk] : 0.0;
    }
  };
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nk) { loadA(s, kb + s * BK); loadB(s, kb + s * BK); }
    cp_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_wait<ST - 2>();
    __syncthreads();
    const int nx = kc + ST - 1;
    if (nx < nk) { loadA(nx % ST, kb + nx * BK); loadB(nx % ST, kb + nx * BK); }
    cp_commit();
    const int buf = kc % ST;
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      const double a = (double)sm.A[buf][r][kk];
#pragma unroll
      for (int i = 0; i < MAXC / 2; ++i)
        if (h + 2 * i < C) acc[i] = fma(a, sm.Bm[buf][kk][h + 2 * i], acc[i]);
    }
  }
  cp_wait<0>();
  __syncthreads();
  // split-K partial tile [BR][C] (fp64) in this CTA's smem, then a DSMEM reduction by rows
  double *part = reinterpret_cast<double *>(dsm1);
#pragma unroll
  for (int i = 0; i < MAXC / 2; ++i)
    if (h + 2 * i < C) part[r * MAXC + h + 2 * i] = acc[i];
  cg::cluster_group cl = cg::this_cluster();
  if (d.S1 > 1) cl.sync(); else __syncthreads();
  const int rows = BR / d.S1, rb = sp * rows;
  for (int e = tid; e < rows * C; e += OP_THREADS) {
    const int rr = rb + e / C, c = e % C;
    double v = 0.0;
    for (int q = 0; q < d.S1; ++q) {
      const double *pp = d.S1 > 1 ? cl.map_shared_rank(part, q) : part;
      v += pp[rr * MAXC + c];
    }
    if (n0 + rr < N) p.b.Um[((size_t)t * N + n0 + rr) * d.Cp + c] = v;
  }
  if (d.S1 > 1) cl.sync();
  return;
}

}  // namespace

cudaError_t launch_mu_stage1(const KParams &p, const double *mu_src, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_mu_stage1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemM1));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1, p.d.nRT1 * p.d.S1, p.d.Tl);
  cfg.blockDim = dim3(OP_THREADS);
  cfg.dynamicSmemBytes = sizeof(SmemM1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = p.d.S1;   // the split-K CTAs of one row tile form a cluster
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_mu_stage1, p, mu_src);
}

}  // namespace cmtcs
