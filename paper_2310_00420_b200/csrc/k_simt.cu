// The batched CG loop of one E-step (Alg. 1, for every task t, cluster c and
// right-hand side of Alg. 2 lines 5-6) with the dense operator on the FP32 CUDA
// cores: op_kind = CMTCS_OP_DENSE_FP32.
//
// Why a second engine: the north_star allows the 3xTF32 tensor-core operator "only if the oracle
// tolerance holds".  tcgen05's fp32 accumulation truncates; over long contractions that shrinks
// |Ad| by a few 1e-7 relative with one sign, which moves the Lanczos log-det ν̄ and hence L(θ̂) by
// more than 1e-3 at configs 4-5.  FFMA rounds to nearest: this engine's errors are
// unbiased, and it is the tolerance-exact path.
//
// Per CG step u (one launch each, stream-ordered; every kernel returns at once when the previous
// update left no column active, so the host checks termination only every few steps):
//   k_simt_probe<1>   U[t][j][n] = Σ_d Φ_t[n][d] · D[t][j][d]                     (probe columns)
//   k_simt_mean1      Um[t][n][c] = Σ_d Φ_t[n][d] · Dm[t][c][d]                  (fp64 mean columns)
//   k_simt_probe<2>   W[t][j][d] = β Σ_n Φ_t[n][d] · U[t][j][n] + α_c ⊙ D, dᵀW partials per 128 rows
//   k_simt_mean2      Wm likewise in fp64, dᵀWm partials
//   k_simt_update     Alg. 1 lines 3-7 per column (γ_u, x, r, ξ_u, d; convergence; transcript)
//
// The probe operator is a 128 × 128 × 8 register-tiled SGEMM (256 threads, 8 × 8 outputs per
// thread, double-buffered shared memory fed from registers): stage 1 multiplies Φ_t (K-major) by the
// directions (K-major); stage 2 reads Φ_t itself as the M-major A operand (no Φᵀ copy) against U.
// Both stages accumulate in fp32 FFMA (round to nearest); the stage-2 epilogue forms
// W = β·acc + α ⊙ d in fp64 from the fp64 α and rounds once, and dᵀW (the same rounded W the residual
// update subtracts) in fp64.  γ_u and ξ_u are fp64 and applied in fp64.
#include <stdlib.h>

#include "cmtcs_internal.cuh"

namespace cmtcs {

namespace {

constexpr int SBM = 128;               // output rows per CTA (n in stage 1, d in stage 2)
constexpr int SBN = 128;               // probe columns per CTA
constexpr int SLD = SBM + 4;           // padded smem row (16-byte aligned rows)
constexpr int STH = 256;
constexpr int MTH = 256;               // mean-column kernels
constexpr int MBK = 16;

__device__ __forceinline__ float4 ldg4(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }
__device__ __forceinline__ float4 ldcs4(const float *p) { return __ldcs(reinterpret_cast<const float4 *>(p)); }

__device__ __forceinline__ bool loop_done(const KParams &p, int u) {
  return u > 0 && *(volatile const int *)(p.b.alive + u - 1) == 0;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- probe operator: U = Φ D (STAGE 1), W = βΦᵀU + α ⊙ D (STAGE 2) -----------------------------
// grid (ceil(P / 128), ceil(M / 128), T_loc); a tile with no active column returns at once.
// Accumulation (TWO): a serial fp32 sum over K = 16384 has a random rounding error ~ε·√K relative
// to the partial sums; the two-level form sums each 64-long block of the contraction in fp32 and
// adds the block sums (round to nearest) into a second accumulator, ~ε·(√64 + √(K/64)).
template <int STAGE, bool TWO>
struct SimtCfg {
  static constexpr int BK = TWO ? 16 : 8;          // contraction slab
  static constexpr int NV = BK / 8;                // float4 of A (and of B) staged per thread and slab
  static constexpr int FLUSH = TWO ? 64 / BK : 0;  // slabs per block sum
  static constexpr int MINB = TWO ? 1 : 2;         // CTAs per SM (register budget 255 / 128)
};

template <int STAGE, bool TWO>
__global__ void __launch_bounds__(STH, SimtCfg<STAGE, TWO>::MINB) k_simt_probe(KParams p, int u) {
  using CF = SimtCfg<STAGE, TWO>;
  constexpr int BK = CF::BK, NV = CF::NV;
  __shared__ __align__(16) float As[2][BK][SLD];
  __shared__ __align__(16) float Bs[2][BK][SLD];
  __shared__ double red[STH / 32][SBN];
  if (loop_done(p, u)) return;
  const Dims &d = p.d;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int t = blockIdx.z, rt = blockIdx.y, j0 = blockIdx.x * SBN, m0 = rt * SBM;
  const int M = STAGE == 1 ? d.N : d.D;      // output rows
  const int KD = STAGE == 1 ? d.D : d.N;     // contraction length (multiple of 4)
  const int ncol = min(SBN, d.P - j0);
  const int *flag = p.b.flag + (size_t)t * d.P + j0;
  if (!__syncthreads_or(tid < ncol && flag[tid] == 1)) return;
  if (STAGE == 2 && rt == 0 && tid == 0) atomicAdd(p.b.histp + u, ncol);
  const float *__restrict__ phi = p.phi + (size_t)t * d.phi_task_stride;
  const float *__restrict__ bsrc = STAGE == 1 ? p.b.D32 + (size_t)t * d.P * d.D : p.b.Uh + (size_t)t * d.Pp * d.N;

  // NV float4 of A and of B per thread and slab, staged in registers across the slab's FMAs.
  // K-major tiles (stage-1 A, both B): rows idx/(BK/4), k quads idx%(BK/4), stored transposed
  // [k][row] (the k quads of a warp fall ≥ 8 banks apart: row stride SLD ≡ 4 mod 32);
  // stage-2 A is Φ itself, M-major: k = idx/32, rows (idx%32)·4, stored as is.
  float4 ra[NV], rb[NV];
  auto gload = [&](int k0) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int idx = tid + v * STH;
      if (STAGE == 1) {
        const int m = m0 + idx / (BK / 4), k = k0 + (idx % (BK / 4)) * 4;
        ra[v] = (m < M && k < KD) ? ldcs4(phi + (size_t)m * d.D + k) : z;
      } else {
        const int k = k0 + (idx >> 5), m = m0 + (idx & 31) * 4;
        ra[v] = (k < KD && m < M) ? ldcs4(phi + (size_t)k * d.D + m) : z;
      }
      const int row = idx / (BK / 4), k = k0 + (idx % (BK / 4)) * 4;
      rb[v] = (row < ncol && k < KD) ? ldg4(bsrc + (size_t)(j0 + row) * KD + k) : z;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int idx = tid + v * STH;
      const int row = idx / (BK / 4), kq = (idx % (BK / 4)) * 4;
      if (STAGE == 1) {
        As[buf][kq + 0][row] = ra[v].x;
        As[buf][kq + 1][row] = ra[v].y;
        As[buf][kq + 2][row] = ra[v].z;
        As[buf][kq + 3][row] = ra[v].w;
      } else {
        *reinterpret_cast<float4 *>(&As[buf][idx >> 5][(idx & 31) * 4]) = ra[v];
      }
      Bs[buf][kq + 0][row] = rb[v].x;
      Bs[buf][kq + 1][row] = rb[v].y;
      Bs[buf][kq + 2][row] = rb[v].z;
      Bs[buf][kq + 3][row] = rb[v].w;
    }
  };

  // acc2[i][h] = outputs (row i, columns 2h, 2h+1): packed FFMA2 (two round-to-nearest fp32 FMAs per
  // instruction, the A value a scalar broadcast operand) halves the issue slots of the math
  float2 acc2[8][4], tot2[TWO ? 8 : 1][TWO ? 4 : 1];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int h = 0; h < 4; ++h) acc2[i][h] = make_float2(0.f, 0.f);
  if (TWO) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int h = 0; h < 4; ++h) tot2[TWO ? i : 0][TWO ? h : 0] = make_float2(0.f, 0.f);
  }
  const int nk = (KD + BK - 1) / BK;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) gload((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 b[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                           make_float2(b1.z, b1.w)};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int h = 0; h < 4; ++h) acc2[i][h] = __ffma2_rn(make_float2(a[i], a[i]), b[h], acc2[i][h]);
    }
    if (TWO && ((kt + 1) % CF::FLUSH == 0 || kt + 1 == nk)) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float2 &tt = tot2[TWO ? i : 0][TWO ? h : 0];
          tt.x += acc2[i][h].x;
          tt.y += acc2[i][h].y;
          acc2[i][h] = make_float2(0.f, 0.f);
        }
    }
    if (kt + 1 < nk) sstore(buf ^ 1);
    __syncthreads();
  }
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 v = TWO ? tot2[TWO ? i : 0][TWO ? h : 0] : acc2[i][h];
      acc[i][2 * h] = v.x;
      acc[i][2 * h + 1] = v.y;
    }

  // acc[i][j]: row m0 + (i < 4 ? ty*4 + i : 64 + ty*4 + i-4), column j0 + (j < 4 ? tx*4 + j : 64 + tx*4 + j-4)
  if (STAGE == 1) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (c >= ncol) continue;
      float *out = p.b.Uh + ((size_t)t * d.Pp + j0 + c) * d.N;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int m = m0 + g * 64 + ty * 4;
        if (m < M) *reinterpret_cast<float4 *>(out + m) =
            make_float4(acc[4 * g][j], acc[4 * g + 1][j], acc[4 * g + 2][j], acc[4 * g + 3][j]);
      }
    }
  } else {
    const double beta = p.beta;
    const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double dot = 0.0;
      const int c = (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (c < ncol) {
        const size_t col = (size_t)t * d.P + j0 + c;
        const double *al = p.b.alpha64 + (size_t)((j0 + c) / d.K) * d.D;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const int m = m0 + g * 64 + ty * 4;
          if (m >= M) continue;
          const float4 dv = *reinterpret_cast<const float4 *>(p.b.D32 + col * d.D + m);
          const double2 a01 = *reinterpret_cast<const double2 *>(al + m);
          const double2 a23 = *reinterpret_cast<const double2 *>(al + m + 2);
          float4 w;
          w.x = (float)fma(beta, (double)acc[4 * g + 0][j], a01.x * (double)dv.x);
          w.y = (float)fma(beta, (double)acc[4 * g + 1][j], a01.y * (double)dv.y);
          w.z = (float)fma(beta, (double)acc[4 * g + 2][j], a23.x * (double)dv.z);
          w.w = (float)fma(beta, (double)acc[4 * g + 3][j], a23.y * (double)dv.w);
          *reinterpret_cast<float4 *>(p.b.W + col * d.D + m) = w;
          dot += (double)dv.x * (double)w.x + (double)dv.y * (double)w.y + (double)dv.z * (double)w.z +
                 (double)dv.w * (double)w.w;
        }
      }
      // dᵀW over this tile's 128 rows: the ty pair inside a warp, then the 8 warps (fixed order)
      dot += __shfl_xor_sync(0xffffffffu, dot, 16);
      if (lane < 16) red[warp][c] = dot;
    }
    __syncthreads();
    if (tid < ncol) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < STH / 32; ++w) s += red[w][tid];
      p.b.dAd[((size_t)t * d.P + j0 + tid) * d.nRT2 + rt] = s;
    }
  }
}

// ---- fp64 mean columns ----------------------------------------------------------------------------
__device__ __forceinline__ bool task_mean_active(const KParams &p, int t) {
  int a = 0;
  for (int c = 0; c < p.d.C; ++c) a |= (p.b.flagm[(size_t)t * p.d.C + c] == 1);
  return a != 0;
}

// Um[t][n][c] = Σ_d Φ_t[n][d] · Dm[t][c][d]; grid (ceil(N/128), T_loc); thread = row n, half the clusters
__global__ void __launch_bounds__(MTH) k_simt_mean1(KParams p, int u) {
  __shared__ __align__(16) float As[MBK][SBM + 1];
  __shared__ double Bm[MBK][MAXC];
  if (loop_done(p, u)) return;
  const Dims &d = p.d;
  const int t = blockIdx.y, tid = threadIdx.x, n0 = blockIdx.x * SBM;
  if (!task_mean_active(p, t)) return;
  const float *__restrict__ phi = p.phi + (size_t)t * d.phi_task_stride;
  const double *__restrict__ dm = p.b.Dm + (size_t)t * d.C * d.D;
  const int r = tid & (SBM - 1), h = tid >> 7;
  double acc[MAXC / 2];
#pragma unroll
  for (int i = 0; i < MAXC / 2; ++i) acc[i] = 0.0;
  for (int k0 = 0; k0 < d.D; k0 += MBK) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i) {   // 128 rows × 16 k, transposed into As[k][row]
      const int idx = tid + i * MTH, row = idx >> 2, kq = (idx & 3) * 4;
      const int n = n0 + row, k = k0 + kq;
      const float4 v = (n < d.N && k < d.D) ? ldcs4(phi + (size_t)n * d.D + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      As[kq][row] = v.x; As[kq + 1][row] = v.y; As[kq + 2][row] = v.z; As[kq + 3][row] = v.w;
    }
    if (tid < MBK * d.C) {
      const int c = tid / MBK, kk = tid % MBK;
      Bm[kk][c] = (k0 + kk < d.D) ? dm[(size_t)c * d.D + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < MBK; ++kk) {
      const double a = (double)As[kk][r];
#pragma unroll
      for (int i = 0; i < MAXC / 2; ++i)
        if (h + 2 * i < d.C) acc[i] = fma(a, Bm[kk][h + 2 * i], acc[i]);
    }
  }
  if (n0 + r < d.N) {
#pragma unroll
    for (int i = 0; i < MAXC / 2; ++i)
      if (h + 2 * i < d.C) p.b.Um[((size_t)t * d.N + n0 + r) * d.Cp + h + 2 * i] = acc[i];
  }
}

// Wm[t][c][d] = β Σ_n Φ_t[n][d] · Um[t][n][c] + α_cd · Dm[t][c][d], dᵀWm partial per 128 rows of d;
// grid (ceil(D/128), T_loc)
__global__ void __launch_bounds__(MTH) k_simt_mean2(KParams p, int u) {
  __shared__ __align__(16) float As[MBK][SBM];
  __shared__ double Bm[MBK][MAXC];
  __shared__ double red[MTH / 32][MAXC / 2];
  if (loop_done(p, u)) return;
  const Dims &d = p.d;
  const int t = blockIdx.y, tid = threadIdx.x, rt = blockIdx.x, d0 = rt * SBM;
  if (!task_mean_active(p, t)) return;
  const float *__restrict__ phi = p.phi + (size_t)t * d.phi_task_stride;
  const double *__restrict__ um = p.b.Um + (size_t)t * d.N * d.Cp;
  const int r = tid & (SBM - 1), h = tid >> 7;
  double acc[MAXC / 2];
#pragma unroll
  for (int i = 0; i < MAXC / 2; ++i) acc[i] = 0.0;
  for (int k0 = 0; k0 < d.N; k0 += MBK) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i) {   // 16 rows of Φ × 128 columns (d): coalesced
      const int idx = tid + i * MTH, kr = idx >> 5, dq = (idx & 31) * 4;
      const int n = k0 + kr, dd = d0 + dq;
      *reinterpret_cast<float4 *>(&As[kr][dq]) =
          (n < d.N && dd < d.D) ? ldcs4(phi + (size_t)n * d.D + dd) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (tid < MBK * d.C) {
      const int kk = tid / d.C, c = tid % d.C;
      Bm[kk][c] = (k0 + kk < d.N) ? um[(size_t)(k0 + kk) * d.Cp + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < MBK; ++kk) {
      const double a = (double)As[kk][r];
#pragma unroll
      for (int i = 0; i < MAXC / 2; ++i)
        if (h + 2 * i < d.C) acc[i] = fma(a, Bm[kk][h + 2 * i], acc[i]);
    }
  }
  const int dd = d0 + r;
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int i = 0; i < MAXC / 2; ++i) {
    const int c = h + 2 * i;
    double v = 0.0;
    if (c < d.C && dd < d.D) {
      const size_t o = ((size_t)t * d.C + c) * d.D + dd;
      const double dv = p.b.Dm[o];
      const double w = fma(p.beta, acc[i], p.b.alpha64[(size_t)c * d.D + dd] * dv);
      p.b.Wm[o] = w;
      v = dv * w;
    }
    v = warp_sum_d(v);
    if (lane == 0) red[warp][i] = v;
  }
  __syncthreads();
  if (tid < d.C) {   // cluster c = h + 2i lives in warps 4h .. 4h+3
    const int c = tid, hh = c & 1, i = c >> 1;
    double s = 0.0;
    for (int w = 0; w < 4; ++w) s += red[4 * hh + w][i];
    p.b.dAdm[((size_t)t * d.C + c) * d.nRT2 + rt] = s;
  }
}

// ---- update (Alg. 1 lines 3-7), one warp per column ---------------------------------------------
__device__ void report_simt(int *status, int code, int t, int col, int u) {
  if (atomicCAS(status, 0, code) == 0) {
    status[1] = t;
    status[2] = col;
    status[3] = u;
  }
}

__device__ void simt_update_probe(const KParams &p, int t, int col, int u, int lane) {
  const Dims &d = p.d;
  const size_t g = (size_t)t * d.P + col;
  double dpart = 0.0;
  for (int i = lane; i < d.nRT2; i += 32) dpart += p.b.dAd[g * d.nRT2 + i];
  const double dAd = warp_sum_d(dpart);
  const double rr = p.b.rr[g];
  if (!(dAd > 0.0)) {  // Alg. 1 line 3 breakdown
    if (lane == 0) {
      report_simt(p.b.status, ST_BREAKDOWN, d.t0 + t, col, u + 1);
      p.b.flag[g] = 0;
    }
    return;
  }
  const double gam = rr / dAd;
  float4 *__restrict__ x4 = reinterpret_cast<float4 *>(p.b.X + g * d.D);
  float4 *__restrict__ r4 = reinterpret_cast<float4 *>(p.b.R + g * d.D);
  float4 *__restrict__ d4 = reinterpret_cast<float4 *>(p.b.D32 + g * d.D);
  const float4 *__restrict__ w4 = reinterpret_cast<const float4 *>(p.b.W + g * d.D);
  const int n4 = d.D >> 2;
  double acc = 0.0;
  for (int i = lane; i < n4; i += 32) {
    const float4 dv = d4[i], wv = w4[i];
    float4 x = x4[i], r = r4[i];
    x.x = (float)fma(gam, (double)dv.x, (double)x.x);
    x.y = (float)fma(gam, (double)dv.y, (double)x.y);
    x.z = (float)fma(gam, (double)dv.z, (double)x.z);
    x.w = (float)fma(gam, (double)dv.w, (double)x.w);
    r.x = (float)fma(-gam, (double)wv.x, (double)r.x);
    r.y = (float)fma(-gam, (double)wv.y, (double)r.y);
    r.z = (float)fma(-gam, (double)wv.z, (double)r.z);
    r.w = (float)fma(-gam, (double)wv.w, (double)r.w);
    x4[i] = x;
    r4[i] = r;
    acc = fma((double)r.x, (double)r.x, acc);
    acc = fma((double)r.y, (double)r.y, acc);
    acc = fma((double)r.z, (double)r.z, acc);
    acc = fma((double)r.w, (double)r.w, acc);
  }
  const double rrn = warp_sum_d(acc);
  const double xi = rrn / rr;
  const bool conv = sqrt(rrn) <= p.tol * sqrt((double)d.D);   // ‖b‖ = ‖p‖ = √D (A5)
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
    for (int i = lane; i < n4; i += 32) {   // this lane's own stores of r: no sync needed
      const float4 r = r4[i];
      float4 dv = d4[i];
      dv.x = (float)fma(xi, (double)dv.x, (double)r.x);
      dv.y = (float)fma(xi, (double)dv.y, (double)r.y);
      dv.z = (float)fma(xi, (double)dv.z, (double)r.z);
      dv.w = (float)fma(xi, (double)dv.w, (double)r.w);
      d4[i] = dv;
    }
  }
}

__device__ void simt_update_mean(const KParams &p, int t, int c, int u, int lane) {
  const Dims &d = p.d;
  const size_t g = (size_t)t * d.C + c;
  double dpart = 0.0;
  for (int i = lane; i < d.nRT2; i += 32) dpart += p.b.dAdm[g * d.nRT2 + i];
  const double dAd = warp_sum_d(dpart);
  const double rr = p.b.rrm[g];
  if (!(dAd > 0.0)) {
    if (lane == 0) {
      report_simt(p.b.status, ST_BREAKDOWN, d.t0 + t, -1 - c, u + 1);
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
  const double rrn = warp_sum_d(acc);
  const double xi = rrn / rr;
  const bool conv = sqrt(rrn) <= p.tol_mean * sqrt(p.b.bnorm2[t]);
  const bool stop = conv || (u + 1 >= d.cap);
  if (lane == 0) {
    p.b.stepsm[g] = u + 1;
    p.b.rrm[g] = rrn;
    if (stop) p.b.flagm[g] = conv ? 0 : 2;
    else atomicAdd(p.b.alive + u, 1);
  }
  if (!stop) {
    for (int i = lane; i < n2; i += 32) {
      const double2 rn = r[i];
      double2 dd = dv[i];
      dd.x = fma(xi, dd.x, rn.x);
      dd.y = fma(xi, dd.y, rn.y);
      dv[i] = dd;
    }
  }
}

__global__ void __launch_bounds__(256) k_simt_update(KParams p, int u) {
  if (loop_done(p, u)) return;
  const Dims &d = p.d;
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.b.u = u + 1;   // CG steps executed
  if (w >= d.Tl * (d.P + d.C)) return;
  const int t = w / (d.P + d.C), j = w % (d.P + d.C);
  const bool active = j < d.P ? p.b.flag[(size_t)t * d.P + j] == 1 : p.b.flagm[(size_t)t * d.C + (j - d.P)] == 1;
  if (!active) return;
  if (lane == 0) {
    if (atomicMax(p.b.tmark + t, u + 1) < u + 1) atomicAdd(p.b.histt + u, 1);   // tasks active at step u
    atomicAdd(j < d.P ? p.b.hist + u : p.b.histm + u, 1);
  }
  if (j < d.P) simt_update_probe(p, t, j, u, lane);
  else simt_update_mean(p, t, j - d.P, u, lane);
}

}  // namespace

// The CG loop of an E-step on the CUDA cores.  Termination is checked on the host every
// SimtTiming::B steps (alive[u] read back through pinned memory); the kernels of steps past the last
// one return at once.  *launches counts the kernels launched; with `tm` the operator (stage 1 → the
// end of stage 2, mean kernels included) and update durations are accumulated from CUDA events.
cudaError_t run_simt_cg(const KParams &p, int *h_alive, int64_t *launches, SimtTiming *tm, cudaStream_t s) {
  const Dims &d = p.d;
  const dim3 g1((d.P + SBN - 1) / SBN, (d.N + SBM - 1) / SBM, d.Tl);
  const dim3 g2((d.P + SBN - 1) / SBN, (d.D + SBM - 1) / SBM, d.Tl);
  const dim3 gm1((d.N + SBM - 1) / SBM, d.Tl), gm2((d.D + SBM - 1) / SBM, d.Tl);
  const int gu = (d.Tl * (d.P + d.C) + 7) / 8;
  constexpr int B = SimtTiming::B;
  const bool two = !getenv("CMTCS_SIMT_ONE");   // experiments: single fp32 accumulator
  cudaError_t e = cudaMemsetAsync(p.b.u, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  auto collect = [&](int n) -> cudaError_t {   // the last n steps' events (their work has completed)
    for (int i = 0; i < n; ++i) {
      float a = 0.f, b2 = 0.f;
      cudaError_t r = cudaEventElapsedTime(&a, tm->ev[3 * i], tm->ev[3 * i + 1]);
      if (r == cudaSuccess) r = cudaEventElapsedTime(&b2, tm->ev[3 * i + 1], tm->ev[3 * i + 2]);
      if (r != cudaSuccess) return r;
      tm->op_ms += a;
      tm->upd_ms += b2;
    }
    return cudaSuccess;
  };
  int pending = 0;
  for (int u = 0; u < d.cap; ++u) {
    const int slot = u % B;
    if (tm) cudaEventRecord(tm->ev[3 * slot], s);
    if (two) k_simt_probe<1, true><<<g1, STH, 0, s>>>(p, u);
    else k_simt_probe<1, false><<<g1, STH, 0, s>>>(p, u);
    k_simt_mean1<<<gm1, MTH, 0, s>>>(p, u);
    if (two) k_simt_probe<2, true><<<g2, STH, 0, s>>>(p, u);
    else k_simt_probe<2, false><<<g2, STH, 0, s>>>(p, u);
    k_simt_mean2<<<gm2, MTH, 0, s>>>(p, u);
    if (tm) cudaEventRecord(tm->ev[3 * slot + 1], s);
    k_simt_update<<<gu, 256, 0, s>>>(p, u);
    if (tm) cudaEventRecord(tm->ev[3 * slot + 2], s);
    *launches += 5;
    ++pending;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (slot == B - 1 || u + 1 == d.cap) {
      e = cudaMemcpyAsync(h_alive, p.b.alive + u, sizeof(int), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e == cudaSuccess && tm) e = collect(pending);
      if (e != cudaSuccess) return e;
      pending = 0;
      if (*h_alive == 0) break;
    }
  }
  return cudaSuccess;
}

}  // namespace cmtcs
