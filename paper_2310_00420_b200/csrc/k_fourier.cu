// The partial-Fourier operator of the paper's own workload (§4): Φ_t = Ω_t F with F the
// unitary DFT and Ω_t a random subset of N of its D rows, real-embedded as [Re(Ω_t F); Im(Ω_t F)]
// (reading F1).  For real v,
//     ΦᵀΦ v = Re(Fᴴ Ω_tᵀΩ_t F v) = DFT⁻¹(m_sym ⊙ DFT(v)) / D,   m_sym(k) = (m(k) + m(−k mod D)) / 2,
// a circulant ("τ_D = O(D log D) ... Fourier operators"), so A = βΦᵀΦ + diag(α) is
// applied with one forward and one inverse FFT of length D per CG step; ΦᵀΦ is never formed.
//
// Design (B200): one CTA runs the whole CG (Alg. 1) of one column at a time, the
// column's vectors x, r, d in registers (D / 512 per thread) and the FFT in shared memory — nothing
// leaves the SM inside the CG loop except the transcript (γ_u, ξ_u).  CTAs are persistent over the
// columns.  The K probe columns per (t, c) run in fp32 (vectors, FFT) with fp64 dot products; the C
// mean columns run the same kernel instantiated in fp64 (μ parity).  The FFT is radix-2:
// a decimation-in-frequency forward pass (natural order in, bit-reversed out), the mask applied in
// bit-reversed order, and a decimation-in-time inverse pass (bit-reversed in, natural out): no
// permutation passes.  Twiddles exp(−2πi k/D) come from a table (fp64 sincospi, rounded once) for the
// stages whose butterfly span is ≥ 64, and are computed with sincospi for the short spans (a table
// read there would be a 16-way bank conflict).
#include <stdio.h>

#include <algorithm>

#include "cmtcs_internal.cuh"

namespace cmtcs {

namespace {

constexpr int FT = 512;                 // threads per CTA
constexpr int FDMAX = 8192;             // largest D (fp64: 128 KB of complex buffer)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <class R> struct C2 { R x, y; };

template <class R>
__device__ __forceinline__ C2<R> cmul(C2<R> a, C2<R> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <class R>
__device__ __forceinline__ C2<R> cmulc(C2<R> a, C2<R> b) {   // a · conj(b)
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
__device__ __forceinline__ void sincospi_(float x, float *s, float *c) { sincospif(x, s, c); }
__device__ __forceinline__ void sincospi_(double x, double *s, double *c) { sincospi(x, s, c); }

// exp(−2πi·pos/(2·half)), pos < half
template <class R>
__device__ __forceinline__ C2<R> twiddle(const C2<R> *tw, int pos, int half, int logD) {
  if (half >= 32) return tw[pos << (logD - __ffs(half))];   // pos · D / (2·half)
  R s, c;
  sincospi_(-(R)pos / (R)half, &s, &c);
  return {c, s};
}

template <class R>
__device__ double block_sum(double v, double *red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();   // red is reused by consecutive reductions
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < FT / 32; ++i) s += red[i];     // fixed order: deterministic
  return s;
}

// Forward DIF DFT (unnormalised, exp(−2πi kd/D)) in place: natural order in, bit-reversed out.
template <class R>
__device__ void fft_dif(C2<R> *buf, const C2<R> *tw, int D, int logD) {
  for (int half = D >> 1; half >= 1; half >>= 1) {
    const int lh = __ffs(half) - 1;
    for (int b = threadIdx.x; b < (D >> 1); b += FT) {
      const int grp = b >> lh, pos = b & (half - 1);
      const int i = (grp << (lh + 1)) + pos, j = i + half;
      const C2<R> a = buf[i], c = buf[j];
      buf[i] = {a.x + c.x, a.y + c.y};
      buf[j] = cmul<R>({a.x - c.x, a.y - c.y}, twiddle<R>(tw, pos, half, logD));
    }
    __syncthreads();
  }
}
// Inverse DIT DFT (unnormalised, exp(+2πi kd/D)) in place: bit-reversed order in, natural out.
template <class R>
__device__ void ifft_dit(C2<R> *buf, const C2<R> *tw, int D, int logD) {
  for (int half = 1; half < D; half <<= 1) {
    const int lh = __ffs(half) - 1;
    for (int b = threadIdx.x; b < (D >> 1); b += FT) {
      const int grp = b >> lh, pos = b & (half - 1);
      const int i = (grp << (lh + 1)) + pos, j = i + half;
      const C2<R> a = buf[i], t = cmulc<R>(buf[j], twiddle<R>(tw, pos, half, logD));
      buf[i] = {a.x + t.x, a.y + t.y};
      buf[j] = {a.x - t.x, a.y - t.y};
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int brev(int k, int logD) { return (int)(__brev((unsigned)k) >> (32 - logD)); }

// Shared memory: buf C2<R>[D] | tw C2<R>[D/2] | msym2 uint8[D] | red double[FT/32] | misc
// (fp32 at D = 8192: 104 KB — two CTAs per SM)
template <class R>
__host__ __device__ constexpr size_t fourier_smem(int D) {
  return (size_t)D * sizeof(C2<R>) + (size_t)(D / 2) * sizeof(C2<R>) + (size_t)D + (FT / 32) * sizeof(double) + 64;
}

// 2·m_sym of task t in bit-reversed order (0, 1 or 2): each sampled row k counts at k and at −k mod D.
// The counts are formed in `scratch` (D ints: the FFT buffer, free between columns).
__device__ void build_mask(const int *rows, int N, int D, int logD, int *scratch, unsigned char *msym2) {
  for (int i = threadIdx.x; i < D; i += FT) scratch[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += FT) {
    const int k = rows[i];
    atomicAdd(scratch + brev(k, logD), 1);
    atomicAdd(scratch + brev((D - k) & (D - 1), logD), 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < D; i += FT) msym2[i] = (unsigned char)scratch[i];
  __syncthreads();
}

// D·ΦᵀΦ d into buf (natural order; Re is the result): the caller forms W = β/D·Re(buf) + α ⊙ d
// entry by entry (no W array: registers).  Each thread first writes only its own entries
// (j = tid + FT·e), which only it reads back after the inverse pass, so no barrier is needed between
// the caller's reads of one application and the writes of the next.
template <class R, int E>
__device__ __forceinline__ void apply_normal(const R (&dv)[E], C2<R> *buf, const C2<R> *tw,
                                             const unsigned char *msym2, int D, int logD) {
#pragma unroll
  for (int e = 0; e < E; ++e) buf[threadIdx.x + FT * e] = {dv[e], (R)0};
  __syncthreads();
  fft_dif<R>(buf, tw, D, logD);
  for (int q = threadIdx.x; q < D; q += FT) {
    const R m = (R)0.5 * (R)msym2[q];
    buf[q] = {buf[q].x * m, buf[q].y * m};
  }
  __syncthreads();
  ifft_dit<R>(buf, tw, D, logD);
}

// b_t = βΦ_tᵀy_t (Eq. 6): Φᵀ[u; w] = Re(Fᴴ Ωᵀ(u + iw)) — the measurements scattered to
// their DFT rows, one inverse DFT, ÷√D.  One CTA per task, fp64.
__global__ void __launch_bounds__(FT) k_fourier_rhs(KParams p) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const Dims &d = p.d;
  const int t = blockIdx.x, D = d.D, N = d.N, logD = __ffs(D) - 1;
  C2<double> *buf = reinterpret_cast<C2<double> *>(fsm);
  C2<double> *tw = buf + D;
  double *red = reinterpret_cast<double *>(tw + D / 2);
  for (int k = threadIdx.x; k < D / 2; k += FT) {
    double s, c;
    sincospi(-2.0 * k / D, &s, &c);
    tw[k] = {c, s};
  }
  for (int i = threadIdx.x; i < D; i += FT) buf[i] = {0.0, 0.0};
  __syncthreads();
  const int *rows = p.rows + (size_t)t * N;
  const float *y = p.y + (size_t)t * 2 * N;
  for (int i = threadIdx.x; i < N; i += FT) buf[brev(rows[i], logD)] = {(double)y[i], (double)y[N + i]};
  __syncthreads();
  ifft_dit<double>(buf, tw, D, logD);
  const double sc = p.beta / sqrt((double)D);
  double nb = 0.0;
  for (int i = threadIdx.x; i < D; i += FT) {
    const double b = sc * buf[i].x;
    p.b.b64[(size_t)t * D + i] = b;
    nb = fma(b, b, nb);
  }
  nb = block_sum<double>(nb, red);
  if (threadIdx.x == 0) p.b.bnorm2[t] = nb;
}

// The CG of Alg. 1 per column, persistent over the columns of one kind: the probe columns (R =
// float, columns (t, c, k) → X, transcript) or the mean columns (R = double, (t, c) → Xm, and
// ‖y_t − Φ_t μ_tc‖² for ℓ, reading A1).
// E = D / FT entries per thread, a template constant so x, r, d live in registers
template <class R, bool MEAN, int E>
__global__ void __launch_bounds__(FT, 1) k_cg_fourier(KParams p) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const Dims &d = p.d;
  const int D = d.D, N = d.N, logD = __ffs(D) - 1;
  C2<R> *buf = reinterpret_cast<C2<R> *>(fsm);
  C2<R> *tw = buf + D;
  unsigned char *msym2 = reinterpret_cast<unsigned char *>(tw + D / 2);
  double *red = reinterpret_cast<double *>(msym2 + D);
  for (int k = threadIdx.x; k < D / 2; k += FT) {
    double s, c;
    sincospi(-2.0 * k / D, &s, &c);
    tw[k] = {(R)c, (R)s};
  }
  const int per_task = MEAN ? d.C : d.P;
  const int ncol = d.Tl * per_task;
  const R betaD = (R)(p.beta / (double)D);
  int mask_t = -1;
  for (int g = blockIdx.x; g < ncol; g += gridDim.x) {
    const int t = g / per_task, j = g % per_task;
    const int c = MEAN ? j : j / d.K, k = MEAN ? 0 : j % d.K;
    if (t != mask_t) {
      build_mask(p.rows + (size_t)t * N, N, D, logD, reinterpret_cast<int *>(buf), msym2);
      mask_t = t;
    }
    R x[E], r[E], dv[E];
    const double *al = p.b.alpha64 + (size_t)c * D + threadIdx.x;   // α_c of this thread's entries
    double rr = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = threadIdx.x + FT * e;
      R v;
      if (MEAN) {
        v = (R)p.b.b64[(size_t)t * D + i];
      } else {
        uint64_t wd;
        if (p.probe_bits) {
          wd = p.probe_bits[(((size_t)t * d.C + c) * d.K + k) * d.nw + (i >> 6)];
        } else {
          const uint64_t wi = ((((uint64_t)p.it * d.T + (uint64_t)(d.t0 + t)) * d.C + c) * d.K + k) * d.nw + (i >> 6);
          wd = mix64(p.seed + (wi + 1ull) * 0x9E3779B97F4A7C15ull);
        }
        v = ((wd >> (i & 63)) & 1ull) ? (R)-1 : (R)1;
      }
      x[e] = (R)0;
      r[e] = v;
      dv[e] = v;
      rr += (double)v * (double)v;
    }
    rr = block_sum<R>(rr, red);
    const double bnorm = sqrt(rr);
    const double tol = MEAN ? p.tol_mean : p.tol;
    int steps = 0, flag = rr > 0.0 ? 1 : 0;   // zero right-hand side: x = 0 in 0 steps (A8)
    for (int u = 0; u < d.cap && flag == 1; ++u) {
      apply_normal<R, E>(dv, buf, tw, msym2, D, logD);
      double dad = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const R w = betaD * buf[threadIdx.x + FT * e].x + (R)__ldg(al + FT * e) * dv[e];
        dad = fma((double)dv[e], (double)w, dad);
      }
      dad = block_sum<R>(dad, red);
      if (!(dad > 0.0)) {   // Alg. 1 line 3 breakdown
        if (threadIdx.x == 0 && atomicCAS(p.b.status, 0, ST_BREAKDOWN) == 0) {
          p.b.status[1] = d.t0 + t;
          p.b.status[2] = MEAN ? -1 - c : j;
          p.b.status[3] = u + 1;
        }
        flag = 0;
        break;
      }
      // γ, ξ: fp64; the probe columns apply them in fp32 and record the applied values (as the dense path)
      const double gam = MEAN ? rr / dad : (double)(float)(rr / dad);
      const R gr = (R)gam;
      double rn = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const R w = betaD * buf[threadIdx.x + FT * e].x + (R)__ldg(al + FT * e) * dv[e];
        x[e] = x[e] + gr * dv[e];
        r[e] = r[e] - gr * w;
        rn = fma((double)r[e], (double)r[e], rn);
      }
      rn = block_sum<R>(rn, red);
      const double xi = MEAN ? rn / rr : (double)(float)(rn / rr);
      if (!MEAN && threadIdx.x == 0) {
        const size_t col = (size_t)t * d.P + j;
        p.b.gam[col * d.cap + u] = gam;
        p.b.xi[col * d.cap + u] = xi;
      }
      if (threadIdx.x == 0) atomicAdd((MEAN ? p.b.histm : p.b.hist) + u, 1);
      rr = rn;
      steps = u + 1;
      const bool conv = sqrt(rn) <= tol * bnorm;
      if (conv) flag = 0;
      else if (u + 1 >= d.cap) flag = 2;
      else {
        const R xr = (R)xi;
#pragma unroll
        for (int e = 0; e < E; ++e) dv[e] = r[e] + xr * dv[e];
      }
    }
    if (MEAN) {
      double *xm = p.b.Xm + ((size_t)t * d.C + c) * D;
#pragma unroll
      for (int e = 0; e < E; ++e) xm[threadIdx.x + FT * e] = (double)x[e];
      // ‖y − Φμ‖² (reading A1): Φμ = [Re; Im] of the DFT of μ at the sampled rows, ÷√D
#pragma unroll
      for (int e = 0; e < E; ++e) buf[threadIdx.x + FT * e] = {x[e], (R)0};
      __syncthreads();
      fft_dif<R>(buf, tw, D, logD);
      const int *rows = p.rows + (size_t)t * N;
      const float *y = p.y + (size_t)t * 2 * N;
      const double isq = 1.0 / sqrt((double)D);
      double res = 0.0;
      for (int i = threadIdx.x; i < N; i += FT) {
        const C2<R> f = buf[brev(rows[i], logD)];
        const double a = (double)y[i] - isq * (double)f.x, b = (double)y[N + i] - isq * (double)f.y;
        res = fma(a, a, fma(b, b, res));
      }
      res = block_sum<R>(res, red);
      if (threadIdx.x == 0) {
        p.b.resm[(size_t)t * d.C + c] = res;
        p.b.stepsm[(size_t)t * d.C + c] = steps;
        p.b.flagm[(size_t)t * d.C + c] = flag;
      }
    } else {
      float *xp = p.b.X + ((size_t)t * d.P + j) * D;
#pragma unroll
      for (int e = 0; e < E; ++e) xp[threadIdx.x + FT * e] = (float)x[e];
      if (threadIdx.x == 0) {
        p.b.steps[(size_t)t * d.P + j] = steps;
        p.b.flag[(size_t)t * d.P + j] = flag;
      }
    }
    __syncthreads();   // buf / msym reuse by the next column
  }
}

}  // namespace

bool fourier_supported(int D, int N, char *why) {
  if (D < FT || D > FDMAX || (D & (D - 1))) {
    snprintf(why, 256, "partial-Fourier operator needs D a power of two in [%d, %d] (got %d)", FT, FDMAX, D);
    return false;
  }
  if (N < 1 || N > D) {
    snprintf(why, 256, "partial-Fourier operator needs 1 <= N <= D sampled rows (got %d)", N);
    return false;
  }
  return true;
}

cudaError_t launch_fourier_rhs(const KParams &p, cudaStream_t s) {
  const size_t sm = fourier_smem<double>(p.d.D);
  cudaError_t e = cudaFuncSetAttribute(k_fourier_rhs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k_fourier_rhs<<<p.d.Tl, FT, sm, s>>>(p);
  return cudaGetLastError();
}

namespace {
template <int E>
cudaError_t launch_fourier_cg_e(const KParams &p, int sms, cudaStream_t s) {
  const size_t sf = fourier_smem<float>(p.d.D), sd = fourier_smem<double>(p.d.D);
  cudaError_t e = cudaFuncSetAttribute(k_cg_fourier<float, false, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_cg_fourier<double, true, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sd);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cg_fourier<float, false, E>, FT, sf);
  if (e != cudaSuccess) return e;
  const int np = p.d.Tl * p.d.P, nm = p.d.Tl * p.d.C;
  const int gp = std::min(np, std::max(1, occ) * sms), gm = std::min(nm, sms);
  k_cg_fourier<float, false, E><<<gp, FT, sf, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_cg_fourier<double, true, E><<<gm, FT, sd, s>>>(p);
  return cudaGetLastError();
}
}  // namespace

// both CG kernels (probe columns fp32, mean columns fp64), persistent over their columns
cudaError_t launch_fourier_cg(const KParams &p, int sms, cudaStream_t s) {
  switch (p.d.D / FT) {
    case 1: return launch_fourier_cg_e<1>(p, sms, s);
    case 2: return launch_fourier_cg_e<2>(p, sms, s);
    case 4: return launch_fourier_cg_e<4>(p, sms, s);
    case 8: return launch_fourier_cg_e<8>(p, sms, s);
    case 16: return launch_fourier_cg_e<16>(p, sms, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cmtcs
