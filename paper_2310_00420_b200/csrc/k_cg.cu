// K2 (right-hand side), K3 (Rademacher probes + CG initialisation) and K4 (fused CG update).
//
// Alg. 1, per column:
//   line 1  x₁ = 0, r₁ = b, d₁ = r₁                               -> k_init_columns
//   line 3  γ_u = r_uᵀr_u / d_uᵀAd_u    (dᵀAd from K1's fp64 partials)
//   line 4  x_{u+1} = x_u + γ_u d_u
//   line 5  r_{u+1} = r_u − γ_u Ad_u
//   line 6  ξ_u = r_{u+1}ᵀr_{u+1} / r_uᵀr_u
//   line 7  d_{u+1} = r_{u+1} + ξ_u d_u                            -> k_update (one CTA per column)
// The transcript (γ_u, ξ_u) of every probe column is kept for the log-det quadrature (Eq. 7).
// A column stops after step u when ‖r_{u+1}‖₂ ≤ tol·‖b‖₂ or u = cap (reading A5).
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

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
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
    for (int i = threadIdx.x; i < d.D; i += blockDim.x) {
      const uint64_t wd = ov ? ov[i >> 6] : probe_word(p.seed, wbase + (uint64_t)(i >> 6));
      const float v = ((wd >> (i & 63)) & 1ull) ? -1.f : 1.f;
      p.b.X[base + i] = 0.f;
      p.b.R[base + i] = v;
      p.b.Dh[base + i] = v;     // ±1 is exact in tf32
      p.b.Dl[base + i] = 0.f;
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

__device__ void report(int *status, int code, int t, int col, int u) {
  if (atomicCAS(status, 0, code) == 0) {
    status[1] = t;
    status[2] = col;
    status[3] = u;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per column (8 columns per CTA): Alg. 1 lines 3-7 with warp-shuffle fp64 dot products.
__global__ void __launch_bounds__(UPD_THREADS) k_update(KParams p) {
  const Dims &d = p.d;
  const int u = *p.b.u;
  if (u >= d.cap) return;
  const int lane = threadIdx.x & 31;
  const int slot = blockIdx.x * (UPD_THREADS / 32) + (threadIdx.x >> 5), t = blockIdx.y;
  const double tol = p.tol;
  if (slot < d.P) {
    // ------------------------------ fp32 probe column ---------------------------------------
    if (slot >= p.b.m_act[t]) return;
    const int col = p.b.act[(size_t)t * d.P + slot];
    const size_t g = (size_t)t * d.P + col;
    double dAd = 0.0;
    for (int i = 0; i < d.nRT2; ++i) dAd += p.b.dAd[g * d.nRT2 + i];
    const double rr = p.b.rr[g];
    if (!(dAd > 0.0)) {  // Alg. 1 line 3 breakdown
      if (lane == 0) {
        report(p.b.status, ST_BREAKDOWN, d.t0 + t, col, u + 1);
        p.b.flag[g] = 0;
      }
      return;
    }
    const double gam = rr / dAd;
    float4 *x4 = reinterpret_cast<float4 *>(p.b.X + g * d.D);
    float4 *r4 = reinterpret_cast<float4 *>(p.b.R + g * d.D);
    float4 *dh4 = reinterpret_cast<float4 *>(p.b.Dh + g * d.D);
    float4 *dl4 = reinterpret_cast<float4 *>(p.b.Dl + g * d.D);
    const float4 *w4 = reinterpret_cast<const float4 *>(p.b.W + g * d.D);
    const int n4 = d.D >> 2;
    double acc = 0.0;
    for (int i = lane; i < n4; i += 32) {
      const float4 dh = dh4[i], dl = dl4[i], wv = w4[i];
      const float4 dv = make_float4(dh.x + dl.x, dh.y + dl.y, dh.z + dl.z, dh.w + dl.w);  // exact
      float4 xv = x4[i], rv = r4[i];
      xv.x = (float)fma(gam, (double)dv.x, (double)xv.x);
      xv.y = (float)fma(gam, (double)dv.y, (double)xv.y);
      xv.z = (float)fma(gam, (double)dv.z, (double)xv.z);
      xv.w = (float)fma(gam, (double)dv.w, (double)xv.w);
      rv.x = (float)fma(-gam, (double)wv.x, (double)rv.x);
      rv.y = (float)fma(-gam, (double)wv.y, (double)rv.y);
      rv.z = (float)fma(-gam, (double)wv.z, (double)rv.z);
      rv.w = (float)fma(-gam, (double)wv.w, (double)rv.w);
      x4[i] = xv;
      r4[i] = rv;
      acc += (double)rv.x * rv.x + (double)rv.y * rv.y + (double)rv.z * rv.z + (double)rv.w * rv.w;
    }
    const double rrn = warp_sum(acc);
    const double xi = rrn / rr;
    const bool conv = sqrt(rrn) <= tol * sqrt((double)d.D);
    const bool stop = conv || (u + 1 >= d.cap);
    if (lane == 0) {
      p.b.gam[g * d.cap + u] = gam;
      p.b.xi[g * d.cap + u] = xi;
      p.b.steps[g] = u + 1;
      p.b.rr[g] = rrn;
      if (stop) p.b.flag[g] = conv ? 0 : 2;
      else atomicAdd(p.b.alive + u, 1);
    }
    if (!stop) {
      for (int i = lane; i < n4; i += 32) {
        const float4 rv = r4[i], dh = dh4[i], dl = dl4[i];
        float4 dv = make_float4(dh.x + dl.x, dh.y + dl.y, dh.z + dl.z, dh.w + dl.w);
        dv.x = (float)fma(xi, (double)dv.x, (double)rv.x);
        dv.y = (float)fma(xi, (double)dv.y, (double)rv.y);
        dv.z = (float)fma(xi, (double)dv.z, (double)rv.z);
        dv.w = (float)fma(xi, (double)dv.w, (double)rv.w);
        // store d_{u+1} as the exact pair (tf32(d), d − tf32(d)) the tensor-core operator reads
        float4 h4;
        h4.x = tf32_rn(dv.x); h4.y = tf32_rn(dv.y); h4.z = tf32_rn(dv.z); h4.w = tf32_rn(dv.w);
        dh4[i] = h4;
        dl4[i] = make_float4(dv.x - h4.x, dv.y - h4.y, dv.z - h4.z, dv.w - h4.w);
      }
    }
  } else if (slot < d.P + d.C) {
    // ------------------------------ fp64 mean column ----------------------------------------
    const int c = slot - d.P;
    const int gi = t * d.C + c;
    if (p.b.flagm[gi] != 1) return;
    const size_t g = (size_t)gi;
    double dAd = 0.0;
    for (int i = 0; i < d.nRT2; ++i) dAd += p.b.dAdm[g * d.nRT2 + i];
    const double rr = p.b.rrm[g];
    if (!(dAd > 0.0)) {
      if (lane == 0) {
        report(p.b.status, ST_BREAKDOWN, d.t0 + t, -1 - c, u + 1);
        p.b.flagm[g] = 0;
      }
      return;
    }
    const double gam = rr / dAd;
    double2 *x = reinterpret_cast<double2 *>(p.b.Xm + g * d.D);
    double2 *r = reinterpret_cast<double2 *>(p.b.Rm + g * d.D);
    double2 *dv = reinterpret_cast<double2 *>(p.b.Dm + g * d.D);
    const double2 *w = reinterpret_cast<const double2 *>(p.b.Wm + g * d.D);
    const int n2 = d.D >> 1;
    double acc = 0.0;
    for (int i = lane; i < n2; i += 32) {
      const double2 dd = dv[i], ww = w[i];
      double2 xx = x[i], rn = r[i];
      xx.x = fma(gam, dd.x, xx.x);
      xx.y = fma(gam, dd.y, xx.y);
      rn.x = fma(-gam, ww.x, rn.x);
      rn.y = fma(-gam, ww.y, rn.y);
      x[i] = xx;
      r[i] = rn;
      acc = fma(rn.x, rn.x, acc);
      acc = fma(rn.y, rn.y, acc);
    }
    const double rrn = warp_sum(acc);
    const double xi = rrn / rr;
    const bool conv = sqrt(rrn) <= p.tol_mean * sqrt(p.b.bnorm2[t]);
    const bool stop = conv || (u + 1 >= d.cap);
    if (lane == 0) {
      p.b.stepsm[g] = u + 1;
      p.b.rrm[g] = rrn;
      if (stop) p.b.flagm[g] = conv ? 0 : 2;
      else atomicAdd(p.b.alive + u, 1);
    }
    if (!stop)
      for (int i = lane; i < n2; i += 32) {
        const double2 rn = r[i];
        double2 dd = dv[i];
        dd.x = fma(xi, dd.x, rn.x);
        dd.y = fma(xi, dd.y, rn.y);
        dv[i] = dd;
      }
  }
  if (threadIdx.x == 0) atomicMax(p.b.ts + 4 * u + 2, globaltimer());
}

// End of one CG step inside the graph's WHILE body: advance the step counter and keep looping
// while some column is still active and the cap is not reached.
__global__ void k_advance(KParams p, cudaGraphConditionalHandle h) {
  const int u = *p.b.u;
  if (u >= p.d.cap) {  // an unrolled body ran past the end: nothing left to do
    cudaGraphSetConditional(h, 0u);
    return;
  }
  const int more = (p.b.alive[u] > 0) && (u + 1 < p.d.cap);
  *p.b.u = more ? u + 1 : p.d.cap;   // u = cap marks "done" for the remaining unrolled steps
  cudaGraphSetConditional(h, more ? 1u : 0u);
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
  return cudaGetLastError();
}

cudaError_t launch_update(const KParams &p, cudaStream_t s) {
  const int per = UPD_THREADS / 32;
  k_update<<<dim3((p.d.P + p.d.C + per - 1) / per, p.d.Tl), UPD_THREADS, 0, s>>>(p);
  return cudaGetLastError();
}

__global__ void k_advance_plain(KParams p) { *p.b.u += 1; }

cudaError_t launch_advance(const KParams &p, unsigned long long cond_handle, cudaStream_t s) {
  if (cond_handle == 0ull) k_advance_plain<<<1, 1, 0, s>>>(p);
  else k_advance<<<1, 1, 0, s>>>(p, (cudaGraphConditionalHandle)cond_handle);
  return cudaGetLastError();
}

cudaError_t launch_probe_words(uint64_t seed, int it, int T, int t0, int Tl, int C, int K, int D,
                               uint64_t *out, cudaStream_t s) {
  k_probe_words<<<1184, 256, 0, s>>>(seed, it, T, t0, Tl, C, K, D, out);
  return cudaGetLastError();
}

}  // namespace cmtcs
