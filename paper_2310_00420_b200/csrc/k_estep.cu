// K6 diagonal estimate (Eq. 5), K7 Lanczos-quadrature log-det (Eq. 7-9), K8 ℓ / q / log-lik
// (Eq. 3), K9/K10 M-step (Eq. 4), K11 readout (Alg. 2 lines 17-20) and step statistics.
#include "cmtcs_internal.cuh"

namespace cmtcs {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double block_sum(double v, double *sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += sh[i];
  return s;
}

// K6: s_tc = (1/K) Σ_k p_k ⊙ x_k   (Eq. 5; Alg. 2 line 7).  Probes are regenerated
// from the counter hash (or the override words) instead of being stored.
__global__ void k_diag(KParams p) {
  const Dims &d = p.d;
  const int dd = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y, t = blockIdx.z;
  if (dd >= d.D) return;
  double acc = 0.0;
  for (int k = 0; k < d.K; ++k) {
    uint64_t wd;
    if (p.probe_bits) {
      wd = p.probe_bits[(((size_t)t * d.C + c) * d.K + k) * d.nw + (dd >> 6)];
    } else {
      const uint64_t w = ((((uint64_t)p.it * d.T + (uint64_t)(d.t0 + t)) * d.C + c) * d.K + k) * d.nw + (dd >> 6);
      wd = mix64(p.seed + (w + 1ull) * 0x9E3779B97F4A7C15ull);
    }
    const double x = (double)(d.ldv ? p.b.X[(size_t)dd * d.ldv + (size_t)t * d.Pp + c * d.K + k]   // FP32 engine
                                    : p.b.X[((size_t)t * d.P + c * d.K + k) * d.D + dd]);
    acc += ((wd >> (dd & 63)) & 1ull) ? -x : x;
  }
  p.b.s[((size_t)t * d.C + c) * d.D + dd] = acc / (double)d.K;
}

// K7: τ = D · Σ_u S̄²_{u,1} log λ̄_u for Γ̄ assembled from (γ, ξ) (Eq. 7-8).
// Σ_u S̄²_{u,1} log λ̄_u is exactly e₁ᵀ log(Γ̄) e₁ (S̄ holds the eigenvectors as rows).
// Instead of a serial eigendecomposition per tridiagonal, one CTA per Γ̄ evaluates it in parallel
// from the Stieltjes representation (for any c > 0, with Σ_u S̄²_{u,1} = 1):
//   e₁ᵀ log(Γ̄) e₁ = log c + ∫_ℝ eˣ [ 1/(c + eˣ) − e₁ᵀ(Γ̄ + eˣ I)⁻¹ e₁ ] dx ,
// where e₁ᵀ(Γ̄ + sI)⁻¹e₁ = 1/q₁(s) comes from the bottom-up continued fraction
//   q_U = a_U + s,  q_u = (a_u + s) − b_u² / q_{u+1}   (all q_u > 0: Γ̄ + sI is SPD),
// and the integral is a trapezoid sum with step h = 0.4 over [log λ_lo − 37, log λ_hi + 37]
// (integrand analytic in |Im x| < π ⇒ error ~ e^{−2π²/h} ≈ 1e-21; tails < e^{−37}).
// λ_hi is the Gershgorin bound; λ_lo ≤ λ_min is found by Sturm counts at λ_hi·2^{−j}.
// Matches numpy.linalg.eigh-based Eq. 8 to ~1e-13 (tests/test_gpu_parity.py).  fp64 throughout.
__global__ void __launch_bounds__(128) k_lanczos(const double *__restrict__ gam, const double *__restrict__ xi,
                                                 const int *__restrict__ steps, int n, int ld, int D,
                                                 double *tau, int *status) {
  extern __shared__ double sm_lz[];
  __shared__ double red[128];
  __shared__ int s_bad, s_j;
  const int g = blockIdx.x, tid = threadIdx.x;
  const int U = steps[g];
  double *a = sm_lz, *b2 = sm_lz + ld;
  const double *ga = gam + (size_t)g * ld, *xa = xi + (size_t)g * ld;
  if (tid == 0) { s_bad = 0; s_j = 1 << 30; }
  __syncthreads();
  if (U < 1 || U > ld) {
    if (tid == 0) {
      tau[g] = nan("");
      if (atomicCAS(status, 0, ST_EIG) == 0) { status[1] = g; status[2] = U; status[3] = -1; }
    }
    return;
  }
  // Eq. 7: a_u = Γ̄_uu,  b_u² = Γ̄²_{u,u+1} = ξ_u / γ_u²
  double ghi = -INFINITY;
  for (int i = tid; i < U; i += blockDim.x) {
    const double gi = ga[i];
    if (!(gi > 0.0) || !isfinite(gi)) s_bad = 1;
    a[i] = 1.0 / gi + (i > 0 ? xa[i - 1] / ga[i - 1] : 0.0);
    b2[i] = (i + 1 < U) ? xa[i] / (gi * gi) : 0.0;
  }
  __syncthreads();
  for (int i = tid; i < U; i += blockDim.x) {
    const double r = a[i] + (i > 0 ? sqrt(b2[i - 1]) : 0.0) + sqrt(b2[i]);
    ghi = fmax(ghi, r);
  }
  red[tid] = ghi;
  __syncthreads();
  for (int o = 64; o; o >>= 1) {
    if (tid < o) red[tid] = fmax(red[tid], red[tid + o]);
    __syncthreads();
  }
  const double hi = red[0];
  __syncthreads();
  if (s_bad || !(hi > 0.0) || !isfinite(hi)) {
    if (tid == 0) {
      tau[g] = nan("");
      if (atomicCAS(status, 0, ST_EIG) == 0) { status[1] = g; status[2] = U; status[3] = -2; }
    }
    return;
  }
  // λ_lo: the largest x_j = hi·2^{−j} with no eigenvalue below it (Sturm count = 0)
  {
    const double x = ldexp(hi, -tid);
    double d = a[U - 1] - x;
    int cnt = d < 0.0;
    for (int i = U - 2; i >= 0; --i) {
      if (d == 0.0) d = -1e-300;
      d = (a[i] - x) - b2[i] / d;
      cnt += d < 0.0;
    }
    if (cnt == 0) atomicMin(&s_j, tid);
  }
  __syncthreads();
  if (s_j >= (1 << 30)) {
    if (tid == 0) {
      tau[g] = nan("");
      if (atomicCAS(status, 0, ST_EIG) == 0) { status[1] = g; status[2] = U; status[3] = -3; }
    }
    return;
  }
  const double lo = ldexp(hi, -s_j);
  const double c = sqrt(lo * hi), h = 0.4;
  const double x0 = log(lo) - 37.0, x1 = log(hi) + 37.0;
  const int nn = (int)ceil((x1 - x0) / h) + 1;
  double acc = 0.0;
  bool bad = false;
  for (int k = tid; k < nn; k += blockDim.x) {
    const double s = exp(x0 + k * h);
    double q = a[U - 1] + s;
    for (int i = U - 2; i >= 0; --i) q = (a[i] + s) - b2[i] / q;
    bad |= !(q > 0.0);
    acc += s * (1.0 / (c + s) - 1.0 / q);
  }
  if (bad) s_bad = 1;
  red[tid] = acc;
  __syncthreads();
  for (int o = 64; o; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  if (tid == 0) {
    if (s_bad || !isfinite(red[0])) {
      tau[g] = nan("");
      if (atomicCAS(status, 0, ST_EIG) == 0) { status[1] = g; status[2] = U; status[3] = -4; }
    } else {
      tau[g] = (double)D * (log(c) + h * red[0]);
    }
  }
}

// K8: ν̄_tc = −(1/K)Σ_k τ_tck (Eq. 9);  ℓ̃_tc = ν̄ + Σ_d log α_cd − β‖y − Φμ‖² − μᵀdiag(α)μ
// (reading A1: PAPER.md:59's ℓ minus the c-independent β‖y‖²);  q_t = softmax(½ℓ̃ + log π)
// (Eq. 3);  log p(y_t|θ̂) = logsumexp(½ℓ̃ + log π) + (N/2) log(β/2π)  (A2).
__global__ void k_estep_finish(KParams p) {
  __shared__ double sh[32];
  __shared__ double s_ell[MAXC];
  const Dims &d = p.d;
  const int t = blockIdx.x, tid = threadIdx.x;
  const double beta = p.beta;
  for (int c = 0; c < d.C; ++c) {
    const double *mu = p.b.Xm + ((size_t)t * d.C + c) * d.D;
    const double *al = p.b.alpha64 + (size_t)c * d.D;
    double quad = 0.0;
    for (int i = tid; i < d.D; i += blockDim.x) quad = fma(al[i] * mu[i], mu[i], quad);
    quad = block_sum(quad, sh);
    double res = 0.0;
    if (d.op != CMTCS_OP_PARTIAL_FOURIER) {
      for (int n = tid; n < d.N; n += blockDim.x) {
        const double rv = (double)p.y[(size_t)t * d.N + n] - p.b.Um[((size_t)t * d.N + n) * d.Cp + c];
        res = fma(rv, rv, res);
      }
      res = block_sum(res, sh);
    } else {
      res = p.b.resm[(size_t)t * d.C + c];   // computed with μ by the partial-Fourier CG kernel
    }
    if (tid == 0) {
      double tsum = 0.0;
      for (int k = 0; k < d.K; ++k) tsum += p.b.tau[(size_t)t * d.P + c * d.K + k];
      const double nu = -tsum / (double)d.K;
      p.b.nu[t * d.C + c] = nu;
      s_ell[c] = nu + p.b.logsum_alpha[c] - beta * res - quad;
      p.b.ell[t * d.C + c] = s_ell[c];
    }
  }
  if (tid == 0) {
    double a[MAXC], mx = -INFINITY;
    for (int c = 0; c < d.C; ++c) {
      a[c] = 0.5 * s_ell[c] + p.b.logpi[c];
      mx = fmax(mx, a[c]);
    }
    bool bad = !isfinite(mx);
    for (int c = 0; c < d.C; ++c) bad |= isnan(a[c]) || (a[c] == INFINITY);
    if (bad) {
      if (atomicCAS(p.b.status, 0, ST_NUMERIC) == 0) { p.b.status[1] = d.t0 + t; p.b.status[2] = -1; p.b.status[3] = -1; }
      for (int c = 0; c < d.C; ++c) p.b.q[t * d.C + c] = nan("");
      p.b.ll[t] = nan("");
      return;
    }
    double se = 0.0;
    for (int c = 0; c < d.C; ++c) se += exp(a[c] - mx);
    for (int c = 0; c < d.C; ++c) p.b.q[t * d.C + c] = exp(a[c] - mx) / se;
    // N real measurements per task (the partial-Fourier operator's real embedding has 2N: reading F1)
    const double nmeas = d.op == CMTCS_OP_PARTIAL_FOURIER ? 2.0 * d.N : (double)d.N;
    p.b.ll[t] = mx + log(se) + 0.5 * nmeas * log(beta / (2.0 * 3.14159265358979323846));
  }
}

__global__ void k_alpha_stats(KParams p) {
  __shared__ double sh[32];
  const int c = blockIdx.x;
  double v = 0.0;
  for (int i = threadIdx.x; i < p.d.D; i += blockDim.x) v += log(p.b.alpha64[(size_t)c * p.d.D + i]);
  v = block_sum(v, sh);
  if (threadIdx.x == 0) p.b.logsum_alpha[c] = v;
}

// K9: Eq. 4 sums over this rank's tasks (fixed task order), plus Σ_t log p(y_t).
//   red[c·D + d] = Σ_t q_tc (μ_tcd² + max(s_tcd, var_floor))   red[C·D + c] = Σ_t q_tc
__global__ void k_mstep_partial(KParams p) {
  const Dims &d = p.d;
  const int dd = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  const double *q = p.q_override ? p.q_override : p.b.q;
  if (dd < d.D) {
    double den = 0.0;
    for (int t = 0; t < d.Tl; ++t) {
      const size_t o = ((size_t)t * d.C + c) * d.D + dd;
      const double mu = p.b.Xm[o];
      den = fma(q[t * d.C + c], fma(mu, mu, fmax(p.b.s[o], p.var_floor)), den);
    }
    p.b.red[(size_t)c * d.D + dd] = den;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double num = 0.0;
    for (int t = 0; t < d.Tl; ++t) num += q[t * d.C + c];
    p.b.red[(size_t)d.C * d.D + c] = num;
  }
  if (blockIdx.x == 0 && c == 0 && threadIdx.x == 32) {
    double ll = 0.0;
    for (int t = 0; t < d.Tl; ++t) ll += p.b.ll[t];
    p.b.red[(size_t)d.C * d.D + d.C] = ll;
  }
}

// K10: α̃_cd = min(num_c / den_cd, α_max); clusters with num_c < empty_eps keep α (A10); with
// learn_pi also log π_c.
__global__ void k_mstep_finish(KParams p) {
  const Dims &d = p.d;
  const int dd = blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  const double num = p.b.red[(size_t)d.C * d.D + c];
  // learned mixture weights (reading P1): π_c = (1/T) Σ_t q_tc, num all-reduced over
  // the ranks' tasks and T the global task count; the next E-step's softmax reads log π
  if (p.learn_pi && dd == 0) p.b.logpi[c] = log(num / (double)d.T);
  if (dd >= d.D) return;
  if (num < p.empty_eps) return;
  const double a = fmin(num / p.b.red[(size_t)c * d.D + dd], p.alpha_max);
  p.b.alpha64[(size_t)c * d.D + dd] = a;
  p.b.alpha32[(size_t)c * d.D + dd] = (float)a;
}

// K11: a_t = argmax_c q_tc (ties → lowest c, A11);  ẑ_t = μ_{t,a_t}
__global__ void k_readout(KParams p, double *recon) {
  const Dims &d = p.d;
  const int t = blockIdx.x;
  __shared__ int s_a;
  if (threadIdx.x == 0) {
    int a = 0;
    double best = p.b.q[t * d.C];
    for (int c = 1; c < d.C; ++c)
      if (p.b.q[t * d.C + c] > best) { best = p.b.q[t * d.C + c]; a = c; }
    s_a = a;
    p.b.assign[t] = a;
  }
  __syncthreads();
  if (recon)
    for (int i = threadIdx.x; i < d.D; i += blockDim.x)
      recon[(size_t)t * d.D + i] = p.b.Xm[((size_t)t * d.C + s_a) * d.D + i];
}

// step statistics for cmtcs_step_info (one CTA)
__global__ void k_stats(KParams p) {
  __shared__ double sh[32];
  const Dims &d = p.d;
  const int tid = threadIdx.x;
  const int np = d.Tl * d.P, nm = d.Tl * d.C;
  double smin = 1e300, smax = 0, ssum = 0, mmin = 1e300, mmax = 0, caph = 0;
  for (int i = tid; i < np; i += blockDim.x) {
    const double s = p.b.steps[i];
    smin = fmin(smin, s); smax = fmax(smax, s); ssum += s; caph += (p.b.flag[i] == 2);
  }
  for (int i = tid; i < nm; i += blockDim.x) {
    const double s = p.b.stepsm[i];
    mmin = fmin(mmin, s); mmax = fmax(mmax, s); caph += (p.b.flagm[i] == 2);
  }
  double h = 0, hm = 0, ht = 0, hp = 0;
  for (int u = tid; u < d.cap; u += blockDim.x) {
    h += p.b.hist[u]; hm += p.b.histm[u]; ht += p.b.histt[u]; hp += p.b.histp[u];
  }
  // min/max via negation trick on sums is not possible; use shared reductions
  __shared__ double red[6][256];
  red[0][tid] = smin; red[1][tid] = smax; red[2][tid] = mmin; red[3][tid] = mmax;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (tid < o) {
      red[0][tid] = fmin(red[0][tid], red[0][tid + o]);
      red[1][tid] = fmax(red[1][tid], red[1][tid + o]);
      red[2][tid] = fmin(red[2][tid], red[2][tid + o]);
      red[3][tid] = fmax(red[3][tid], red[3][tid + o]);
    }
    __syncthreads();
  }
  ssum = block_sum(ssum, sh);
  caph = block_sum(caph, sh);
  h = block_sum(h, sh);
  hm = block_sum(hm, sh);
  ht = block_sum(ht, sh);
  hp = block_sum(hp, sh);
  if (tid == 0) {
    double *o = p.b.stats;
    o[0] = np ? red[0][0] : 0; o[1] = red[1][0]; o[2] = np ? ssum / np : 0;
    o[3] = nm ? red[2][0] : 0; o[4] = red[3][0]; o[5] = caph;
    o[6] = h; o[7] = hm; o[8] = ht; o[9] = hp;
  }
}

__global__ void k_copy_transcript(KParams p, double *gam, double *xi) {
  const Dims &d = p.d;
  const size_t n = (size_t)d.Tl * d.P * d.cap;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t col = i / d.cap, u = i % d.cap;
    const bool valid = (int)u < p.b.steps[col];
    if (gam) gam[i] = valid ? p.b.gam[i] : nan("");
    if (xi) xi[i] = valid ? p.b.xi[i] : nan("");
  }
}

}  // namespace

cudaError_t launch_diag(const KParams &p, cudaStream_t s) {
  k_diag<<<dim3((p.d.D + 255) / 256, p.d.C, p.d.Tl), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_lanczos(const double *gam, const double *xi, const int *steps, int n, int ld, int D,
                           double *tau, double *scratch, int *status, cudaStream_t s) {
  (void)scratch;
  if (n <= 0) return cudaSuccess;
  const size_t smem = 2 * (size_t)ld * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_lanczos, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_lanczos<<<n, 128, smem, s>>>(gam, xi, steps, n, ld, D, tau, status);
  return cudaGetLastError();
}

cudaError_t launch_estep_finish(const KParams &p, cudaStream_t s) {
  k_estep_finish<<<p.d.Tl, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_alpha_stats(const KParams &p, cudaStream_t s) {
  k_alpha_stats<<<p.d.C, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_mstep_partial(const KParams &p, cudaStream_t s) {
  k_mstep_partial<<<dim3((p.d.D + 255) / 256, p.d.C), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_mstep_finish(const KParams &p, cudaStream_t s) {
  k_mstep_finish<<<dim3((p.d.D + 255) / 256, p.d.C), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_stats(const KParams &p, cudaStream_t s) {
  k_stats<<<1, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_readout(const KParams &p, double *recon, cudaStream_t s) {
  k_readout<<<p.d.Tl, 256, 0, s>>>(p, recon);
  return cudaGetLastError();
}

cudaError_t launch_copy_transcript(const KParams &p, double *gam, double *xi, cudaStream_t s) {
  k_copy_transcript<<<592, 256, 0, s>>>(p, gam, xi);
  return cudaGetLastError();
}

}  // namespace cmtcs
