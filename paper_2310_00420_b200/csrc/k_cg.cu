// K2 (right-hand side b = βΦᵀy, Eq. 6) and K3 (Rademacher probes, Alg. 2 line 5
// PAPER.md:107, + CG initialisation x₁ = 0, r₁ = d₁ = b, Alg. 1 line 1 PAPER.md:89).
// Lines 3-7 of Alg. 1 (the CG update, K4) run inside the persistent CG kernel, k_cg_persistent.cu.
#include "cmtcs_internal.cuh"

namespace cmtcs {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// word(w) = mix64(seed + (w+1)·φ64)   (reading A6; the splitmix64 sequence started at `seed`)
__device__ __forceinline__ uint64_t probe_word(uint64_t seed, uint64_t w) {
  return mix64(seed + (w + 1ull) * 0x9E3779B97F4A7C15ull);
}

__device__ __forceinline__ double block_sum(double v, double *sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += sh[i];  // fixed order: deterministic
  return s;
}

__global__ void k_rhs(KParams p) {
  // b_t = β Φ_tᵀ y_t in fp64 (Eq. 6)
  const Dims &d = p.d;
  const int t = blockIdx.y, dd = blockIdx.x * blockDim.x + threadIdx.x;
  if (dd >= d.D) return;
  const float *phi = p.phi + (size_t)t * d.phi_task_stride;
  const float *y = p.y + (size_t)t * d.N;
  double acc = 0.0;
  for (int n = 0; n < d.N; ++n) acc = fma((double)phi[(size_t)n * d.D + dd], (double)y[n], acc);
  p.b.b64[(size_t)t * d.D + dd] = p.beta * acc;
}

__global__ void k_bnorm(KParams p) {
  __shared__ double sh[32];
  const Dims &d = p.d;
  const int t = blockIdx.x;
  double v = 0.0;
  for (int i = threadIdx.x; i < d.D; i += blockDim.x) {
    const double b = p.b.b64[(size_t)t * d.D + i];
    v = fma(b, b, v);
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) p.b.bnorm2[t] = v;
}

__global__ void k_init_columns(KParams p) {
  const Dims &d = p.d;
  const int slot = blockIdx.x, t = blockIdx.y;
  if (slot < d.P) {
    // K3: p_{it,t,c,k} ∈ {±1}^D (Alg. 2 line 5) and x₁ = 0, r₁ = d₁ = p (Alg. 1 line 1)
    const int c = slot / d.K, k = slot % d.K;
    const size_t base = ((size_t)t * d.P + slot) * d.D;
    const uint64_t wbase = ((((uint64_t)p.it * d.T + (uint64_t)(d.t0 + t)) * d.C + c) * d.K + k) * d.nw;
    const uint64_t *ov = p.probe_bits ? p.probe_bits + (((size_t)t * d.C + c) * d.K + k) * d.nw : nullptr;
    // (the FP32 engine's d-major probe vectors are written by its own kernel, k_simt.cu)
    for (int i = threadIdx.x; i < d.D && !d.ldv; i += blockDim.x) {
      const uint64_t wd = ov ? ov[i >> 6] : probe_word(p.seed, wbase + (uint64_t)(i >> 6));
      const float v = ((wd >> (i & 63)) & 1ull) ? -1.f : 1.f;
      p.b.X[base + i] = 0.f;
      p.b.R[base + i] = v;
      p.b.D32[base + i] = v;
      if (p.b.Dh) {             // the tensor-core operator's B operand (absent for the FP32 engine)
        p.b.Dh[base + i] = v;   // ±1 is exact in tf32
        p.b.Dl[base + i] = 0.f;
      }
    }
    if (threadIdx.x == 0) {
      const size_t g = (size_t)t * d.P + slot;
      if (g == 0) *p.b.u = 0;
      p.b.rr[g] = (double)d.D;  // ‖p‖² = D exactly
      p.b.flag[g] = 1;
      p.b.steps[g] = 0;
    }
  } else {
    const int c = slot - d.P;
    const size_t base = ((size_t)t * d.C + c) * d.D;
    const double *b = p.b.b64 + (size_t)t * d.D;
    for (int i = threadIdx.x; i < d.D; i += blockDim.x) {
      const double v = b[i];
      p.b.Xm[base + i] = 0.0;
      p.b.Rm[base + i] = v;
      p.b.Dm[base + i] = v;
    }
    if (threadIdx.x == 0) {
      const int g = t * d.C + c;
      p.b.rrm[g] = p.b.bnorm2[t];
      p.b.flagm[g] = p.b.bnorm2[t] > 0.0 ? 1 : 0;  // zero RHS: μ = 0 in 0 steps (A8)
      p.b.stepsm[g] = 0;
    }
  }
}

// K3 for the FP32 engine's d-major probe vectors ([D][T_loc·Pp], column g = t·Pp + j): the same
// probes (reading A6) written coalesced along the columns; padding columns j ≥ P are zeroed
__global__ void k_init_probes_dmajor(KParams p) {
  const Dims &d = p.d;
  const size_t n = (size_t)d.D * d.ldv;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / d.ldv), g = (int)(e % d.ldv);
    const int t = g / d.Pp, j = g % d.Pp;
    float v = 0.f;
    if (j < d.P) {
      const int c = j / d.K, k = j % d.K;
      const uint64_t wbase = ((((uint64_t)p.it * d.T + (uint64_t)(d.t0 + t)) * d.C + c) * d.K + k) * d.nw;
      const uint64_t wd = p.probe_bits ? p.probe_bits[(((size_t)t * d.C + c) * d.K + k) * d.nw + (i >> 6)]
                                       : probe_word(p.seed, wbase + (uint64_t)(i >> 6));
      v = ((wd >> (i & 63)) & 1ull) ? -1.f : 1.f;
    }
    p.b.X[e] = 0.f;
    p.b.R[e] = v;
    p.b.D32[e] = v;
  }
}

__global__ void k_probe_words(uint64_t seed, int it, int T, int t0, int Tl, int C, int K, int D,
                              uint64_t *out) {
  const int nw = (D + 63) / 64;
  const size_t n = (size_t)Tl * C * K * nw;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t w = i % nw, col = i / nw;
    const size_t k = col % K, c = (col / K) % C, tl = col / ((size_t)K * C);
    const uint64_t wb = ((((uint64_t)it * T + (uint64_t)(t0 + tl)) * C + c) * K + k) * nw + w;
    out[i] = probe_word(seed, wb);
  }
}

}  // namespace

cudaError_t launch_rhs(const KParams &p, cudaStream_t s) {
  k_rhs<<<dim3((p.d.D + 255) / 256, p.d.Tl), 256, 0, s>>>(p);
  k_bnorm<<<p.d.Tl, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_init_columns(const KParams &p, cudaStream_t s) {
  k_init_columns<<<dim3(p.d.P + p.d.C, p.d.Tl), 256, 0, s>>>(p);
  if (p.d.ldv) k_init_probes_dmajor<<<4 * 148, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_probe_words(uint64_t seed, int it, int T, int t0, int Tl, int C, int K, int D,
                               uint64_t *out, cudaStream_t s) {
  k_probe_words<<<1184, 256, 0, s>>>(seed, it, T, t0, Tl, C, K, D, out);
  return cudaGetLastError();
}

}  // namespace cmtcs
