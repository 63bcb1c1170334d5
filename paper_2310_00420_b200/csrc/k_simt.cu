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
// The probe operator is a 128 × 128 register-tiled SGEMM (256 threads, 8 × 8 outputs per thread,
// a 4-stage cp.async ring of 16-k slabs): stage 1 multiplies Φ_t (K-major) by the
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
// Both stages are one GEMM shape, C[j][m] = Σ_k A[k][m] · B[j][k]: A is M-major — stage 1 reads
// Φᵀ (transposed once at init, [D][N]), stage 2 reads Φ itself — and B is K-major (the directions'
// or U's rows).
//
// Operands stream through a KST-stage cp.async ring of 16-k slabs (no register staging: the copies
// are in flight for KST − 1 slabs of FMAs).  The M-major A slab (16 k × 128 m) is stored as is; a
// thread reads its rows' float4 at each k, and consecutive rows form the register pairs of packed
// FFMA2 (two round-to-nearest fp32 FMAs per instruction, the B value a scalar broadcast operand).
// The K-major B slab keeps its global layout: row r holds its 16 k as four 16-byte quads at quad
// position q ^ ((r >> 3) & 3) of a 20-float row (16-byte group 5r + quad mod 8), so that the 16
// threads of a half-warp reading rows 4·tx + j at one k quad hit all 8 bank groups twice (two
// wavefronts per 256 bytes, the minimum; the unswizzled row hits 4 groups); a thread reads a float4
// of 4 consecutive k per row.
//
// Accumulation: a serial fp32 sum over K = 16384 has a random rounding error ~ε·√K relative to the
// partial sums; each 64-long block of the contraction is summed in fp32 and the block sums are added
// (round to nearest) into a second accumulator, ~ε·(√64 + √(K/64)).
constexpr int KBK = 16;                    // k per slab
constexpr int KST = 4;                     // ring stages
constexpr int KLD = 20;                    // K-major smem row (16 k + 4 pad), floats
constexpr int FLUSH = 64 / KBK;            // slabs per block sum

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ int kq_phys(int row, int q) { return q ^ ((row >> 3) & 3); }

struct SimtSmem {
  float a[KST][KBK * SLD];                 // M-major A slabs [k][m]
  float b[KST][SBN * KLD];                 // K-major B slabs [j][k] (swizzled quads)
};

// VAR (experiments): 0 = FFMA2 + two-level sums (1 CTA / SM); 1 = scalar FFMA + two-level;
// 2 = FFMA2, single-level sums, 2 CTAs / SM (≤ 128 registers)
template <int STAGE, int VAR>
__global__ void __launch_bounds__(STH, VAR == 2 ? 2 : 1) k_simt_probe(KParams p, int u) {
  constexpr bool TWO = VAR != 2;
  extern __shared__ __align__(16) unsigned char simt_raw[];
  SimtSmem &sm = *reinterpret_cast<SimtSmem *>(simt_raw);
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
  // A[k][m]: stage 1 Φᵀ_t [D][N], stage 2 Φ_t [N][D]; row length M
  const float *__restrict__ amat = STAGE == 1 ? p.b.PT + (size_t)t * d.phi_task_stride
                                              : p.phi + (size_t)t * d.phi_task_stride;
  const float *__restrict__ bsrc = STAGE == 1 ? p.b.D32 + (size_t)t * d.P * d.D : p.b.Uh + (size_t)t * d.Pp * d.N;
  const uint32_t sa0 = (uint32_t)__cvta_generic_to_shared(&sm.a[0][0]);
  const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(&sm.b[0][0]);

  // slab kt → ring slot kt % KST: 2 × 16-byte copies per thread and operand
  auto issue = [&](int kt) {
    const int slot = kt % KST, k0 = kt * KBK;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int idx = tid + v * STH;
      {                                         // A: k row idx/32, 4 m at (idx%32)·4
        const int kr = idx >> 5, c4 = (idx & 31) * 4, k = k0 + kr, m = m0 + c4;
        const bool ok = k < KD && m < M;
        cp_async16(sa0 + 4u * (uint32_t)(slot * KBK * SLD + kr * SLD + c4), ok ? amat + (size_t)k * M + m : amat, ok);
      }
      const int r = idx >> 2, q = idx & 3, k = k0 + 4 * q;   // B: column r of the tile, k quad q
      const bool ok = r < ncol && k < KD;
      cp_async16(sb0 + 4u * (uint32_t)(slot * SBN * KLD + r * KLD + 4 * kq_phys(r, q)),
                 ok ? bsrc + (size_t)(j0 + r) * KD + k : bsrc, ok);
    }
  };

  // acc2[ip][j]: rows (2ip, 2ip+1) of this thread's 8 (ty·4 + i, i < 4; 64 + ty·4 + i − 4), column j
  // of its 8 (tx·4 + j, j < 4; 64 + tx·4 + j − 4)
  float2 acc2[4][8], tot2[TWO ? 4 : 1][TWO ? 8 : 1];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      acc2[i][j] = make_float2(0.f, 0.f);
      if (TWO) tot2[TWO ? i : 0][TWO ? j : 0] = make_float2(0.f, 0.f);
    }
  const int nk = (KD + KBK - 1) / KBK;
#pragma unroll
  for (int s = 0; s < KST - 1; ++s) {
    if (s < nk) issue(s);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<KST - 2>();
    __syncthreads();                            // slab kt landed for all; slot (kt − 1) % KST is free
    if (kt + KST - 1 < nk) issue(kt + KST - 1);
    cp_commit();
    const int slot = kt % KST;
    const float *As = sm.a[slot], *Bs = sm.b[slot];
#pragma unroll
    for (int q = 0; q < 4; ++q) {               // 4 k per step
      float4 bq[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
        bq[j] = *reinterpret_cast<const float4 *>(Bs + r * KLD + 4 * kq_phys(r, q));
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4 lo = *reinterpret_cast<const float4 *>(As + (4 * q + e) * SLD + ty * 4);
        const float4 hi = *reinterpret_cast<const float4 *>(As + (4 * q + e) * SLD + 64 + ty * 4);
        const float2 ap[4] = {make_float2(lo.x, lo.y), make_float2(lo.z, lo.w), make_float2(hi.x, hi.y),
                              make_float2(hi.z, hi.w)};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float bv = reinterpret_cast<const float *>(&bq[j])[e];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (VAR == 1) {
              acc2[i][j].x = fmaf(ap[i].x, bv, acc2[i][j].x);
              acc2[i][j].y = fmaf(ap[i].y, bv, acc2[i][j].y);
            } else {
              acc2[i][j] = __ffma2_rn(ap[i], make_float2(bv, bv), acc2[i][j]);
            }
          }
        }
      }
    }
    if (TWO && ((kt + 1) % FLUSH == 0 || kt + 1 == nk)) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          tot2[TWO ? i : 0][TWO ? j : 0].x += acc2[i][j].x;
          tot2[TWO ? i : 0][TWO ? j : 0].y += acc2[i][j].y;
          acc2[i][j] = make_float2(0.f, 0.f);
        }
    }
  }
  cp_wait<0>();
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float2 v = TWO ? tot2[TWO ? i : 0][TWO ? j : 0] : acc2[i][j];
      acc[2 * i][j] = v.x;
      acc[2 * i + 1][j] = v.y;
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
  cudaError_t e = cudaSuccess;
  static int var = -1;   // dynamic shared memory above 48 KB (one process per GPU); CMTCS_SIMT_VAR experiments
  if (var < 0) {
    var = getenv("CMTCS_SIMT_VAR") ? atoi(getenv("CMTCS_SIMT_VAR")) : 0;
    if (var < 0 || var > 2) var = 0;
    const int sb = (int)sizeof(SimtSmem);
    e = cudaFuncSetAttribute(k_simt_probe<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
    if (e != cudaSuccess) return e;
  }
  e = cudaMemsetAsync(p.b.u, 0, sizeof(int), s);
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
    if (var == 0) k_simt_probe<1, 0><<<g1, STH, sizeof(SimtSmem), s>>>(p, u);
    else if (var == 1) k_simt_probe<1, 1><<<g1, STH, sizeof(SimtSmem), s>>>(p, u);
    else k_simt_probe<1, 2><<<g1, STH, sizeof(SimtSmem), s>>>(p, u);
    k_simt_mean1<<<gm1, MTH, 0, s>>>(p, u);
    if (var == 0) k_simt_probe<2, 0><<<g2, STH, sizeof(SimtSmem), s>>>(p, u);
    else if (var == 1) k_simt_probe<2, 1><<<g2, STH, sizeof(SimtSmem), s>>>(p, u);
    else k_simt_probe<2, 2><<<g2, STH, sizeof(SimtSmem), s>>>(p, u);
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
