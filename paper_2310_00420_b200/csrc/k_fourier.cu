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
#include <stdlib.h>

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

// Twiddles exp(−2πi·pos/(2·half)) stored per stage, tw2[half + pos] (half = 1, 2, ..., D/2; D
// entries): the butterflies of a stage read consecutive entries (a strided single table is a 32-way
// bank conflict at spans 64 .. D/8)
template <class R>
__device__ __forceinline__ C2<R> twiddle(const C2<R> *tw2, int pos, int half) { return tw2[half + pos]; }
template <class R>
__device__ __forceinline__ C2<R> twiddle_g(const double2 *tw2, int pos, int half) {
  const double2 v = __ldg(tw2 + half + pos);
  return {(R)v.x, (R)v.y};
}
// The FFT buffer is padded by one element every 32 (index e → e + e/32): the short-span stages'
// butterfly partners then fall in different banks
__device__ __forceinline__ int pad(int e) { return e + (e >> 5); }

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

template <class R, bool TG>
__device__ __forceinline__ C2<R> tw_at(const C2<R> *tw, const double2 *twg, int pos, int half) {
  return TG ? twiddle_g<R>(twg, pos, half) : twiddle<R>(tw, pos, half);
}
template <class R>
__device__ __forceinline__ C2<R> cadd(C2<R> a, C2<R> b) { return {a.x + b.x, a.y + b.y}; }
template <class R>
__device__ __forceinline__ C2<R> csub(C2<R> a, C2<R> b) { return {a.x - b.x, a.y - b.y}; }

// Forward DIF DFT (unnormalised, exp(−2πi kd/D)) in place: natural order in, bit-reversed out.
// Radix-4 passes (each = two radix-2 DIF stages, written to the same positions, so the output order
// is the radix-2 algorithm's), a final radix-2 stage when log₂D is odd.  With W = exp(−2πi/4q) and
// x₀..x₃ at base + {0, q, 2q, 3q}:  A = x₀ + x₂, B = x₀ − x₂, C = x₁ + x₃, E = x₁ − x₃;
//   out₀ = A + C,  out₁ = (A − C)·W^{2p},  out₂ = (B − iE)·W^p,  out₃ = (B + iE)·W^{3p}.
// TG: twiddles from the shared table (fp32) or the global one (fp64).
template <class R, bool TG>
__device__ void fft_dif(C2<R> *buf, const C2<R> *tw, const double2 *twg, int D) {
  int span = D;
  for (; span >= 4; span >>= 2) {
    const int q = span >> 2, lq = __ffs(q) - 1;
    for (int bf = threadIdx.x; bf < (D >> 2); bf += FT) {
      const int grp = bf >> lq, pos = bf & (q - 1);
      const int base = (grp << (lq + 2)) + pos;
      const int i0 = pad(base), i1 = pad(base + q), i2 = pad(base + 2 * q), i3 = pad(base + 3 * q);
      const C2<R> x0 = buf[i0], x1 = buf[i1], x2 = buf[i2], x3 = buf[i3];
      const C2<R> w1 = tw_at<R, TG>(tw, twg, pos, 2 * q), w2 = tw_at<R, TG>(tw, twg, pos, q);
      const C2<R> w3 = cmul<R>(w1, w2);
      const C2<R> A = cadd<R>(x0, x2), B = csub<R>(x0, x2), Cc = cadd<R>(x1, x3), E = csub<R>(x1, x3);
      buf[i0] = cadd<R>(A, Cc);
      buf[i1] = cmul<R>(csub<R>(A, Cc), w2);
      buf[i2] = cmul<R>({B.x + E.y, B.y - E.x}, w1);   // B − iE
      buf[i3] = cmul<R>({B.x - E.y, B.y + E.x}, w3);   // B + iE
    }
    __syncthreads();
  }
  if (span == 2) {   // log₂D odd: one radix-2 stage of span 2 (twiddle 1)
    for (int bf = threadIdx.x; bf < (D >> 1); bf += FT) {
      const int i = pad(2 * bf), j = pad(2 * bf + 1);
      const C2<R> a = buf[i], c = buf[j];
      buf[i] = cadd<R>(a, c);
      buf[j] = csub<R>(a, c);
    }
    __syncthreads();
  }
}
// Inverse DIT DFT (unnormalised, exp(+2πi kd/D)) in place: bit-reversed order in, natural out — the
// exact reverse: a radix-2 stage of span 2 first when log₂D is odd, then radix-4 passes; with
// c₁ = conj(W^p), c₂ = conj(W^{2p}):  u₀,₁ = x₀ ± x₁c₂,  u₂,₃ = x₂ ± x₃c₂;
//   out₀,₂ = u₀ ± u₂c₁,  out₁,₃ = u₁ ± i·u₃c₁.
template <class R, bool TG>
__device__ void ifft_dit(C2<R> *buf, const C2<R> *tw, const double2 *twg, int D) {
  int span = 4;
  if ((__ffs(D) - 1) & 1) {
    for (int bf = threadIdx.x; bf < (D >> 1); bf += FT) {
      const int i = pad(2 * bf), j = pad(2 * bf + 1);
      const C2<R> a = buf[i], c = buf[j];
      buf[i] = cadd<R>(a, c);
      buf[j] = csub<R>(a, c);
    }
    __syncthreads();
    span = 8;
  }
  for (; span <= D; span <<= 2) {
    const int q = span >> 2, lq = __ffs(q) - 1;
    for (int bf = threadIdx.x; bf < (D >> 2); bf += FT) {
      const int grp = bf >> lq, pos = bf & (q - 1);
      const int base = (grp << (lq + 2)) + pos;
      const int i0 = pad(base), i1 = pad(base + q), i2 = pad(base + 2 * q), i3 = pad(base + 3 * q);
      const C2<R> x0 = buf[i0], x1 = buf[i1], x2 = buf[i2], x3 = buf[i3];
      const C2<R> w1 = tw_at<R, TG>(tw, twg, pos, 2 * q), w2 = tw_at<R, TG>(tw, twg, pos, q);
      const C2<R> t1 = cmulc<R>(x1, w2), t3 = cmulc<R>(x3, w2);
      const C2<R> u0 = cadd<R>(x0, t1), u1 = csub<R>(x0, t1), u2 = cadd<R>(x2, t3), u3 = csub<R>(x2, t3);
      const C2<R> v = cmulc<R>(u2, w1), z = cmulc<R>(u3, w1);
      const C2<R> iz = {-z.y, z.x};
      buf[i0] = cadd<R>(u0, v);
      buf[i2] = csub<R>(u0, v);
      buf[i1] = cadd<R>(u1, iz);
      buf[i3] = csub<R>(u1, iz);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int brev(int k, int logD) { return (int)(__brev((unsigned)k) >> (32 - logD)); }

// Shared memory: buf C2<R>[D + D/32] (padded) | tw2 C2<float>[D] (fp32 only; fp64 reads the global
// table) | msym2 uint8[D] | red double[FT/32] | misc
template <class R>
__host__ __device__ constexpr size_t fourier_smem(int D) {
  return (size_t)(D + D / 32) * sizeof(C2<R>) + (sizeof(R) == 4 ? (size_t)D * sizeof(C2<float>) : 0) + (size_t)D +
         (FT / 32) * sizeof(double) + 64;
}

// the per-stage twiddle table tw2[h + pos] = exp(−2πi·pos/(2h)), fp64 (sincospi), once per context
__global__ void k_fourier_twiddles(double2 *tw2, int D) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < D; e += gridDim.x * blockDim.x) {
    if (e == 0) { tw2[0] = make_double2(1.0, 0.0); continue; }
    const int h = 1 << (31 - __clz(e)), pos = e - h;   // e = h + pos with pos < h
    double sn, cs;
    sincospi(-(double)pos / (double)h, &sn, &cs);
    tw2[e] = make_double2(cs, sn);
  }
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
template <class R, bool TG, int E>
__device__ __forceinline__ void apply_normal(const R (&dv)[E], C2<R> *buf, const C2<R> *tw, const double2 *twg,
                                             const unsigned char *msym2, int D) {
#pragma unroll
  for (int e = 0; e < E; ++e) buf[pad(threadIdx.x + FT * e)] = {dv[e], (R)0};
  __syncthreads();
  fft_dif<R, TG>(buf, tw, twg, D);
  for (int q = threadIdx.x; q < D; q += FT) {
    const R m = (R)0.5 * (R)msym2[q];
    const int qq = pad(q);
    buf[qq] = {buf[qq].x * m, buf[qq].y * m};
  }
  __syncthreads();
  ifft_dit<R, TG>(buf, tw, twg, D);
}

// b_t = βΦ_tᵀy_t (Eq. 6): Φᵀ[u; w] = Re(Fᴴ Ωᵀ(u + iw)) — the measurements scattered to
// their DFT rows, one inverse DFT, ÷√D.  One CTA per task, fp64.
__global__ void __launch_bounds__(FT) k_fourier_rhs(KParams p) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const Dims &d = p.d;
  const int t = blockIdx.x, D = d.D, N = d.N, logD = __ffs(D) - 1;
  C2<double> *buf = reinterpret_cast<C2<double> *>(fsm);
  double *red = reinterpret_cast<double *>(buf + D + D / 32);
  const double2 *twg = reinterpret_cast<const double2 *>(p.b.ftw);
  for (int i = threadIdx.x; i < D + D / 32; i += FT) buf[i] = {0.0, 0.0};
  __syncthreads();
  const int *rows = p.rows + (size_t)t * N;
  const float *y = p.y + (size_t)t * 2 * N;
  for (int i = threadIdx.x; i < N; i += FT) buf[pad(brev(rows[i], logD))] = {(double)y[i], (double)y[N + i]};
  __syncthreads();
  ifft_dit<double, true>(buf, nullptr, twg, D);
  const double sc = p.beta / sqrt((double)D);
  double nb = 0.0;
  for (int i = threadIdx.x; i < D; i += FT) {
    const double b = sc * buf[pad(i)].x;
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
  constexpr bool TG = sizeof(R) == 8;   // fp64: twiddles from the global table (shared memory is full)
  C2<R> *buf = reinterpret_cast<C2<R> *>(fsm);
  C2<R> *tw = buf + D + D / 32;
  unsigned char *msym2 = reinterpret_cast<unsigned char *>(TG ? (void *)tw : (void *)(tw + D));
  double *red = reinterpret_cast<double *>(msym2 + D);
  const double2 *twg = reinterpret_cast<const double2 *>(p.b.ftw);
  if (!TG)
    for (int k = threadIdx.x; k < D; k += FT) {
      const double2 v = twg[k];
      tw[k] = {(R)v.x, (R)v.y};
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
      apply_normal<R, TG, E>(dv, buf, tw, twg, msym2, D);
      double dad = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const R w = betaD * buf[pad(threadIdx.x + FT * e)].x + (R)__ldg(al + FT * e) * dv[e];
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
        const R w = betaD * buf[pad(threadIdx.x + FT * e)].x + (R)__ldg(al + FT * e) * dv[e];
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
      for (int e = 0; e < E; ++e) buf[pad(threadIdx.x + FT * e)] = {x[e], (R)0};
      __syncthreads();
      fft_dif<R, TG>(buf, tw, twg, D);
      const int *rows = p.rows + (size_t)t * N;
      const float *y = p.y + (size_t)t * 2 * N;
      const double isq = 1.0 / sqrt((double)D);
      double res = 0.0;
      for (int i = threadIdx.x; i < N; i += FT) {
        const C2<R> f = buf[pad(brev(rows[i], logD))];
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

// Two probe columns per CTA (fp32): ΦᵀΦ is a real operator with a real symmetric symbol, so one
// complex transform of d₀ + i·d₁ gives ΦᵀΦd₀ (real part) and ΦᵀΦd₁ (imaginary part) — half the FFT
// work per column.  The directions live in shared memory (dsm, the FFT's input), x and r in
// registers; a column that stops keeps d = 0, so it adds nothing to its partner's transform.
__device__ __forceinline__ void block_sum2(double &a, double &b, double *red) {
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = a;
    red[FT / 32 + (threadIdx.x >> 5)] = b;
  }
  __syncthreads();
  a = 0.0;
  b = 0.0;
#pragma unroll
  for (int i = 0; i < FT / 32; ++i) {   // fixed order: deterministic
    a += red[i];
    b += red[FT / 32 + i];
  }
}

template <int E>
__global__ void __launch_bounds__(FT, 1) k_cg_fourier_pair(KParams p) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const Dims &d = p.d;
  const int D = d.D, N = d.N, logD = __ffs(D) - 1;
  C2<float> *buf = reinterpret_cast<C2<float> *>(fsm);
  C2<float> *tw = buf + D + D / 32;
  float *dsm = reinterpret_cast<float *>(tw + D);              // [2][D]
  unsigned char *msym2 = reinterpret_cast<unsigned char *>(dsm + 2 * D);
  double *red = reinterpret_cast<double *>(msym2 + D);        // [2][FT/32]
  const double2 *twg = reinterpret_cast<const double2 *>(p.b.ftw);
  for (int k = threadIdx.x; k < D; k += FT) {
    const double2 v = twg[k];
    tw[k] = {(float)v.x, (float)v.y};
  }
  const int npair = (d.P + 1) / 2;
  const int nwork = d.Tl * npair;
  const float betaD = (float)(p.beta / (double)D);
  int mask_t = -1;
  for (int g = blockIdx.x; g < nwork; g += gridDim.x) {
    const int t = g / npair, j0 = 2 * (g % npair);
    const bool has1 = j0 + 1 < d.P;
    if (t != mask_t) {
      build_mask(p.rows + (size_t)t * N, N, D, logD, reinterpret_cast<int *>(buf), msym2);
      mask_t = t;
    }
    float x[2][E], r[2][E];
    const double *al[2];
    double rr[2] = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = j0 + q, c = j / d.K, k = j % d.K;
      al[q] = p.b.alpha64 + (size_t)min(c, d.C - 1) * D + threadIdx.x;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = threadIdx.x + FT * e;
        float v = 0.f;
        if (q == 0 || has1) {
          uint64_t wd;
          if (p.probe_bits) {
            wd = p.probe_bits[(((size_t)t * d.C + c) * d.K + k) * d.nw + (i >> 6)];
          } else {
            const uint64_t wi = ((((uint64_t)p.it * d.T + (uint64_t)(d.t0 + t)) * d.C + c) * d.K + k) * d.nw + (i >> 6);
            wd = mix64(p.seed + (wi + 1ull) * 0x9E3779B97F4A7C15ull);
          }
          v = ((wd >> (i & 63)) & 1ull) ? -1.f : 1.f;
        }
        x[q][e] = 0.f;
        r[q][e] = v;
        dsm[q * D + i] = v;
        rr[q] += (double)v * (double)v;
      }
    }
    block_sum2(rr[0], rr[1], red);
    const double bnorm[2] = {sqrt(rr[0]), sqrt(rr[1])};
    int steps[2] = {0, 0}, flag[2] = {1, has1 ? 1 : 0};
    for (int u = 0; u < d.cap && (flag[0] == 1 || flag[1] == 1); ++u) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = threadIdx.x + FT * e;
        buf[pad(i)] = {dsm[i], dsm[D + i]};
      }
      __syncthreads();
      fft_dif<float, false>(buf, tw, twg, D);
      for (int q2 = threadIdx.x; q2 < D; q2 += FT) {
        const float m = 0.5f * (float)msym2[q2];
        const int qq = pad(q2);
        buf[qq] = {buf[qq].x * m, buf[qq].y * m};
      }
      __syncthreads();
      ifft_dit<float, false>(buf, tw, twg, D);
      double dad[2] = {0.0, 0.0};
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = threadIdx.x + FT * e;
        const C2<float> b = buf[pad(i)];
        const float d0 = dsm[i], d1 = dsm[D + i];
        const float w0 = betaD * b.x + (float)__ldg(al[0] + FT * e) * d0;
        const float w1 = betaD * b.y + (float)__ldg(al[1] + FT * e) * d1;
        dad[0] = fma((double)d0, (double)w0, dad[0]);
        dad[1] = fma((double)d1, (double)w1, dad[1]);
      }
      block_sum2(dad[0], dad[1], red);
      float gr[2];
      double gam[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        gam[q] = 0.0;
        gr[q] = 0.f;
        if (flag[q] != 1) continue;
        if (!(dad[q] > 0.0)) {   // Alg. 1 line 3 breakdown
          if (threadIdx.x == 0 && atomicCAS(p.b.status, 0, ST_BREAKDOWN) == 0) {
            p.b.status[1] = d.t0 + t;
            p.b.status[2] = j0 + q;
            p.b.status[3] = u + 1;
          }
          flag[q] = 0;
          continue;
        }
        gam[q] = (double)(float)(rr[q] / dad[q]);   // applied in fp32, recorded as applied
        gr[q] = (float)gam[q];
      }
      double rn[2] = {0.0, 0.0};
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = threadIdx.x + FT * e;
        const C2<float> b = buf[pad(i)];
        const float d0 = dsm[i], d1 = dsm[D + i];
        const float w0 = betaD * b.x + (float)__ldg(al[0] + FT * e) * d0;
        const float w1 = betaD * b.y + (float)__ldg(al[1] + FT * e) * d1;
        x[0][e] += gr[0] * d0;
        r[0][e] -= gr[0] * w0;
        x[1][e] += gr[1] * d1;
        r[1][e] -= gr[1] * w1;
        rn[0] = fma((double)r[0][e], (double)r[0][e], rn[0]);
        rn[1] = fma((double)r[1][e], (double)r[1][e], rn[1]);
      }
      block_sum2(rn[0], rn[1], red);
      float xr[2] = {0.f, 0.f};
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (flag[q] != 1) continue;
        const double xi = (double)(float)(rn[q] / rr[q]);
        xr[q] = (float)xi;
        if (threadIdx.x == 0) {
          const size_t col = (size_t)t * d.P + j0 + q;
          p.b.gam[col * d.cap + u] = gam[q];
          p.b.xi[col * d.cap + u] = xi;
          atomicAdd(p.b.hist + u, 1);
        }
        rr[q] = rn[q];
        steps[q] = u + 1;
        if (sqrt(rn[q]) <= p.tol * bnorm[q]) flag[q] = 0;
        else if (u + 1 >= d.cap) flag[q] = 2;
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {   // d = r + ξd for a running column; 0 for a stopped one
        const int i = threadIdx.x + FT * e;
        dsm[i] = flag[0] == 1 ? r[0][e] + xr[0] * dsm[i] : 0.f;
        dsm[D + i] = flag[1] == 1 ? r[1][e] + xr[1] * dsm[D + i] : 0.f;
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (q == 1 && !has1) continue;
      float *xp = p.b.X + ((size_t)t * d.P + j0 + q) * D;
#pragma unroll
      for (int e = 0; e < E; ++e) xp[threadIdx.x + FT * e] = x[q][e];
      if (threadIdx.x == 0) {
        p.b.steps[(size_t)t * d.P + j0 + q] = steps[q];
        p.b.flag[(size_t)t * d.P + j0 + q] = flag[q];
      }
    }
    __syncthreads();   // buf / dsm / msym reuse by the next pair
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
  k_fourier_twiddles<<<(p.d.D + 255) / 256, 256, 0, s>>>(reinterpret_cast<double2 *>(p.b.ftw), p.d.D);
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
  const int gm = std::min(nm, sms);
  if (!getenv("CMTCS_FOURIER_SINGLE")) {   // two probe columns per CTA (one complex transform)
    const size_t s2 = (size_t)(p.d.D + p.d.D / 32) * 8 + (size_t)p.d.D * 8 + (size_t)2 * p.d.D * 4 + p.d.D + 2 * (FT / 32) * 8 + 64;
    e = cudaFuncSetAttribute(k_cg_fourier_pair<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
    if (e != cudaSuccess) return e;
    const int npairs = p.d.Tl * ((p.d.P + 1) / 2);
    k_cg_fourier_pair<E><<<std::min(npairs, sms), FT, s2, s>>>(p);
  } else {
    const int gp = std::min(np, std::max(1, occ) * sms);
    k_cg_fourier<float, false, E><<<gp, FT, sf, s>>>(p);
  }
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
