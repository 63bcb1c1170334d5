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
//   k_simt_mean<1>    Um[t][n][c] = Σ_d Φ_t[n][d] · Dm[t][c][d]                  (fp64 mean columns)
//   k_simt_probe<2>   W[t][j][d] = β Σ_n Φ_t[n][d] · U[t][j][n] + α_c ⊙ D, dᵀW partials per 128 rows
//   k_simt_mean<2>    Wm likewise in fp64, dᵀWm partials
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
constexpr int MBK = 16;
constexpr int MTH = 128;               // mean-column kernels (co-resident with a probe-SGEMM CTA)

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
// Layout (Dims::ldv): the FP32 engine keeps its probe vectors d-major — X, R, D32, W as [D][T_loc·Pp]
// and U as [N][T_loc·Pp], column g = t·Pp + j — so that a k-slab of either operand is 16 contiguous
// rows: both GEMM stages are C[g][m] = Σ_k A[k][m] · B[k][g] with A M-major (stage 1: Φᵀ [D][N],
// transposed once at init; stage 2: Φ itself) and B N-major (the directions, U).
// grid (column tiles, ceil(M / 128), T_loc); a tile with no active column returns at once.
//
// Operands stream through a KST-stage cp.async ring of 32-k slabs [k][128 + 4 pad] (no register
// staging: the copies are in flight for KST − 1 slabs of FMAs).  Per k a thread reads two float4
// of A (its 8 rows) and two of B (its 8 columns) — the 16 distinct float4 of a half-warp are 256
// contiguous bytes, conflict-free — and the next k's four are loaded before this k's FMAs (register
// double buffering).  The FMAs are packed FFMA2: consecutive rows are register pairs, the B value a
// scalar broadcast operand; 32 FFMA2 per k per thread.
//
// Accumulation: a serial fp32 sum over K = 16384 has a random rounding error ~ε·√K relative to the
// partial sums; each 64-long block of the contraction is summed in fp32 and the block sums are added
// (round to nearest) into a second accumulator, ~ε·(√64 + √(K/64)).
//
// (Measured alternatives, C4 32 tasks, ms per EM iteration: this form 1462; 512 threads with 4 × 8
// outputs each, ≤ 128 registers, 4 warps per scheduler: 1614.)
//
// pflat > 0 (shared Φ, P % 4 == 0): the columns of all tasks form one GEMM of pflat = T_loc·P columns
// (one A for everyone), so a task's last partial column tile is not padded — config 5's P = 320
// would otherwise multiply 384 columns per task.
// SMT = true (default): 16-k slabs, 2 stages, the block-sum totals in shared memory (thread-private
// float4 slots, conflict-free), ≤ 128 registers and 106 KB: 2 CTAs per SM, so one CTA's barrier,
// prologue and epilogue overlap the other's FMAs; SMT = false (CMTCS_SIMT_SMT=0): 32-k slabs, 4
// stages, the totals in registers (210 registers: 1 CTA per SM)
template <bool SMT>
struct PCfg {
  static constexpr int KBK = SMT ? 16 : 32;  // k per slab
  static constexpr int KST = SMT ? 2 : 4;    // ring stages
  static constexpr int FLUSH = 64 / KBK;     // slabs per block sum
  static constexpr int MINB = SMT ? 2 : 1;
  static constexpr size_t RING = (size_t)KST * 2 * KBK * SLD * sizeof(float);
  static constexpr size_t SMEM = RING + (SMT ? 64 * STH * sizeof(float) : 0);
};

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }


template <int STAGE, bool SMT>
__global__ void __launch_bounds__(STH, PCfg<SMT>::MINB) k_simt_probe(KParams p, int u, int pflat) {
  using CF = PCfg<SMT>;
  constexpr int KBK = CF::KBK, KST = CF::KST, FLUSH = CF::FLUSH;
  extern __shared__ __align__(16) unsigned char simt_raw[];
  float *ring = reinterpret_cast<float *>(simt_raw);   // [KST][A slab | B slab], slab [KBK][SLD]
  float4 *tot4 = reinterpret_cast<float4 *>(simt_raw + CF::RING);   // SMT: [16][STH] block-sum totals
  __shared__ double red[STH / 32][SBN];
  if (loop_done(p, u)) return;
  const Dims &d = p.d;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int t = blockIdx.z + p.toff, rt = blockIdx.y, j0 = blockIdx.x * SBN, m0 = rt * SBM;
  const int M = STAGE == 1 ? d.N : d.D;      // output rows
  const int KD = STAGE == 1 ? d.D : d.N;     // contraction length (multiple of 4)
  // active-column compaction: this tile multiplies the 4-column groups [32·x, 32·x + 32) of its column
  // space's list of groups with an active column (k_simt_groups): a tile ends up with retired
  // columns only inside a partly active group.  Column space: a task's P columns (d-major base
  // t·Pp, state base t·P), or all tasks' (flat: one space, bases 0).
  const int space = pflat > 0 ? 0 : t, ncs = pflat > 0 ? pflat : d.P;
  const int nlist = p.b.m_act[space];
  if (j0 >= 4 * nlist) return;                   // CTA-uniform
  const int ngrp = min(SBN / 4, nlist - j0 / 4);
  __shared__ int sgrp[SBN / 4];
  if (tid < SBN / 4) sgrp[tid] = tid < ngrp ? p.b.act[(size_t)space * d.Pp / 4 * (pflat > 0 ? d.Tl : 1) + j0 / 4 + tid] : 0;
  __syncthreads();
  const int ncol = 4 * ngrp;                     // multiplied columns of this tile (chunks of 4)
  const size_t gb = pflat > 0 ? 0 : (size_t)t * d.Pp;   // the space's base in the d-major arrays
  const size_t fb = pflat > 0 ? 0 : (size_t)t * d.P;    // ... in the per-column state
  if (STAGE == 2 && rt == 0 && tid == 0) atomicAdd(p.b.histp + u, SBN);   // columns multiplied
  // A[k][m]: stage 1 Φᵀ_t [D][N], stage 2 Φ_t [N][D] (row length M); B[k][g]: D32 [D][ldv] / U [N][ldv]
  const float *__restrict__ amat = STAGE == 1 ? p.b.PT + (size_t)t * d.phi_task_stride
                                              : p.phi + (size_t)t * d.phi_task_stride;
  const float *__restrict__ bmat = (STAGE == 1 ? p.b.D32 : p.b.Uh) + gb;   // + 4·group per chunk
  const size_t ldv = (size_t)d.ldv;
  const uint32_t sa0 = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t sb0 = sa0 + 4u * (uint32_t)(KBK * SLD);

  // slab kt → ring slot kt % KST: KBK/8 16-byte copies per thread and operand (k row idx/32, 4
  // entries at (idx%32)·4)
  auto issue = [&](int kt) {
    const int slot = kt % KST, k0 = kt * KBK;
#pragma unroll
    for (int v = 0; v < KBK / 8; ++v) {
      const int idx = tid + v * STH, kr = idx >> 5, c4 = (idx & 31) * 4, k = k0 + kr;
      const uint32_t so = 4u * (uint32_t)(slot * 2 * KBK * SLD + kr * SLD + c4);
      const bool oka = k < KD && m0 + c4 < M;
      cp_async16(sa0 + so, oka ? amat + (size_t)k * M + m0 + c4 : amat, oka);
      const bool okb = k < KD && c4 < ncol;    // chunk c4/4 = group sgrp[c4/4] (its padding columns too)
      cp_async16(sb0 + so, okb ? bmat + (size_t)k * ldv + 4 * sgrp[c4 >> 2] : bmat, okb);
    }
  };

  // acc2[ip][j]: rows (2ip, 2ip+1) of this thread's 8 (ty·4 + i, i < 4; 64 + ty·4 + i − 4), column j
  // of its 8 (tx·4 + j, j < 4; 64 + tx·4 + j − 4)
  float2 acc2[4][8], tot2[SMT ? 1 : 4][SMT ? 1 : 8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      acc2[i][j] = make_float2(0.f, 0.f);
      if (!SMT) tot2[SMT ? 0 : i][SMT ? 0 : j] = make_float2(0.f, 0.f);
    }
  if (SMT) {
#pragma unroll
    for (int q = 0; q < 16; ++q) tot4[q * STH + tid] = make_float4(0.f, 0.f, 0.f, 0.f);
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
    const float *As = ring + slot * 2 * KBK * SLD + ty * 4, *Bs = ring + (slot * 2 + 1) * KBK * SLD + tx * 4;
    float4 a0 = *reinterpret_cast<const float4 *>(As), a1 = *reinterpret_cast<const float4 *>(As + 64);
    float4 b0 = *reinterpret_cast<const float4 *>(Bs), b1 = *reinterpret_cast<const float4 *>(Bs + 64);
#pragma unroll
    for (int kk = 0; kk < KBK; ++kk) {
      float4 na0, na1, nb0, nb1;
      if (kk + 1 < KBK) {                       // next k's operands before this k's FMAs
        na0 = *reinterpret_cast<const float4 *>(As + (kk + 1) * SLD);
        na1 = *reinterpret_cast<const float4 *>(As + (kk + 1) * SLD + 64);
        nb0 = *reinterpret_cast<const float4 *>(Bs + (kk + 1) * SLD);
        nb1 = *reinterpret_cast<const float4 *>(Bs + (kk + 1) * SLD + 64);
      }
      const float2 ap[4] = {make_float2(a0.x, a0.y), make_float2(a0.z, a0.w), make_float2(a1.x, a1.y),
                            make_float2(a1.z, a1.w)};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      // (column-major order: consecutive FFMA2 share the scalar B operand; row-pair-major, sharing the
      // 64-bit A pair, measured 1.6 % slower)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc2[i][j] = __ffma2_rn(ap[i], make_float2(bv[j], bv[j]), acc2[i][j]);
      if (kk + 1 < KBK) {
        a0 = na0; a1 = na1; b0 = nb0; b1 = nb1;
      }
    }
    if ((kt + 1) % FLUSH == 0 || kt + 1 == nk) {
      if (SMT) {                                // totals in shared memory (thread-private float4 slots)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            float4 tt = tot4[(i * 4 + h) * STH + tid];
            tt.x += acc2[i][2 * h].x;
            tt.y += acc2[i][2 * h].y;
            tt.z += acc2[i][2 * h + 1].x;
            tt.w += acc2[i][2 * h + 1].y;
            tot4[(i * 4 + h) * STH + tid] = tt;
            acc2[i][2 * h] = acc2[i][2 * h + 1] = make_float2(0.f, 0.f);
          }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            tot2[SMT ? 0 : i][SMT ? 0 : j].x += acc2[i][j].x;
            tot2[SMT ? 0 : i][SMT ? 0 : j].y += acc2[i][j].y;
            acc2[i][j] = make_float2(0.f, 0.f);
          }
      }
    }
  }
  cp_wait<0>();
  float2 fin[4][8];                             // the totals
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      if (SMT) {
        const float4 tt = tot4[(i * 4 + h) * STH + tid];
        fin[i][2 * h] = make_float2(tt.x, tt.y);
        fin[i][2 * h + 1] = make_float2(tt.z, tt.w);
      } else {
        fin[i][2 * h] = tot2[SMT ? 0 : i][SMT ? 0 : 2 * h];
        fin[i][2 * h + 1] = tot2[SMT ? 0 : i][SMT ? 0 : 2 * h + 1];
      }
    }

  // outputs: rows m0 + g·64 + ty·4 + r (g, r < 2, 4) = fin[2g + r/2][·].{x|y}; columns
  // j0 + h·64 + tx·4 + q (h, q < 2, 4) = fin[·][4h + q]
  if (STAGE == 1) {                             // U [N][ldv]
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + g * 64 + ty * 4 + r;
        if (m >= M) continue;
        const int ip = 2 * g + r / 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c4 = h * 64 + tx * 4;
          if (c4 >= ncol) continue;
          float4 o;
          o.x = (r & 1) ? fin[ip][4 * h + 0].y : fin[ip][4 * h + 0].x;
          o.y = (r & 1) ? fin[ip][4 * h + 1].y : fin[ip][4 * h + 1].x;
          o.z = (r & 1) ? fin[ip][4 * h + 2].y : fin[ip][4 * h + 2].x;
          o.w = (r & 1) ? fin[ip][4 * h + 3].y : fin[ip][4 * h + 3].x;
          *reinterpret_cast<float4 *>(p.b.Uh + (size_t)m * ldv + gb + 4 * sgrp[c4 >> 2]) = o;
        }
      }
  } else {                                      // W = βΦᵀU + α ⊙ d (fp64, one rounding), dᵀW partials
    const double beta = p.beta;
    const int warp = tid >> 5, lane = tid & 31;
    // α of the tile's 128 rows for every cluster, staged in the (now idle) ring: a thread's 8 columns
    // × 8 rows would otherwise be 64 scalar global loads
    double *sal = reinterpret_cast<double *>(ring);
    __syncthreads();                            // every warp is done with the ring
    for (int e = tid; e < d.C * SBM; e += STH) {
      const int c = e / SBM, r = e % SBM;
      sal[e] = m0 + r < M ? p.b.alpha64[(size_t)c * d.D + m0 + r] : 0.0;
    }
    __syncthreads();
    double dot[8];
    const double *al[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      dot[q] = 0.0;
      const int c = (q >> 2) * 64 + tx * 4 + (q & 3);
      const int jc = min(4 * sgrp[min(c, ncol - 1) >> 2] + (c & 3), ncs - 1);   // column in the space
      al[q] = sal + (size_t)(((fb + jc) % d.P) / d.K) * SBM - m0;                 // the column's cluster
    }
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + g * 64 + ty * 4 + r;
        if (m >= M) continue;
        const int ip = 2 * g + r / 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c4 = h * 64 + tx * 4;
          if (c4 >= ncol) continue;
          const size_t o = (size_t)m * ldv + gb + 4 * sgrp[c4 >> 2];
          const float4 dv = *reinterpret_cast<const float4 *>(p.b.D32 + o);
          const float dq[4] = {dv.x, dv.y, dv.z, dv.w};
          float wq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float acc = (r & 1) ? fin[ip][4 * h + q].y : fin[ip][4 * h + q].x;
            wq[q] = (float)fma(beta, (double)acc, al[4 * h + q][m] * (double)dq[q]);
            dot[4 * h + q] += (double)dq[q] * (double)wq[q];
          }
          *reinterpret_cast<float4 *>(p.b.W + o) = make_float4(wq[0], wq[1], wq[2], wq[3]);
        }
      }
    // dᵀW over this tile's 128 rows: the ty pair inside a warp, then the 8 warps (fixed order)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double v = dot[q] + __shfl_xor_sync(0xffffffffu, dot[q], 16);
      if (lane < 16) red[warp][(q >> 2) * 64 + tx * 4 + (q & 3)] = v;
    }
    __syncthreads();
    const int jt = tid < ncol ? 4 * sgrp[tid >> 2] + (tid & 3) : ncs;   // this thread's column, if real
    if (jt < ncs) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < STH / 32; ++w) s += red[w][tid];
      p.b.dAd[(fb + jt) * d.nRT2 + rt] = s;
    }
  }
}

// 4-warp form (default): the same 128 × 128 tile with 128 threads, 16 rows × 8 columns per thread
// (64 FFMA2 per 6 shared loads per k, against 32 per 4 in the 8-warp form above: the FMA pipe, not
// the issue slots or the shared-memory pipe, paces it), ≤ 255 registers, 2 CTAs per SM; block sums of
// 128 k and running copy pointers by default (VAR = 3 below, DESIGN.md §4/§5).  Thread
// (tx = tid % 16, ty = tid / 16, ty < 8): rows ty·4 + i + 32·g (g, i < 4), columns tx·4 + q + 64·h
// (h < 2, q < 4).  The two-level block sums as above: totals in 32 thread-private float4 slots.
constexpr int QTH = 128;
constexpr int QKBK = 16, QKST = 2;
constexpr size_t QRING = (size_t)QKST * 2 * QKBK * SLD * sizeof(float);
constexpr size_t QSMEM = QRING + (size_t)32 * QTH * sizeof(float4);

// VAR (measured variants, CMTCS_SIMT_VAR): bit 0 — block sums of 128 k instead of 64 (half the
// flushes; ε·(√128 + √(K/128))); bit 1 — copy addresses as running pointers with the
// k-bound test only on the last slab; bit 2 — the block-sum adds as packed FADD2; bit 3 — block sums of 256 k (only as VAR = 11 or 14).
template <int STAGE, int VAR = 0>
__global__ void __launch_bounds__(QTH, 2) k_simt_probe4(KParams p, int u, int pflat) {
  constexpr int KBK = QKBK, KST = QKST, FLUSH = ((VAR & 8) ? 256 : (VAR & 1) ? 128 : 64) / KBK;
  constexpr bool LEAN = (VAR & 2) != 0;
  extern __shared__ __align__(16) unsigned char simt_raw[];
  float *ring = reinterpret_cast<float *>(simt_raw);   // [KST][A slab | B slab], slab [KBK][SLD]
  float4 *tot4 = reinterpret_cast<float4 *>(simt_raw + QRING);   // [32][QTH] block-sum totals
  __shared__ double red[QTH / 32][SBN];
  if (loop_done(p, u)) return;
  const Dims &d = p.d;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int t = blockIdx.z + p.toff, rt = blockIdx.y, j0 = blockIdx.x * SBN, m0 = rt * SBM;
  const int M = STAGE == 1 ? d.N : d.D;      // output rows
  const int KD = STAGE == 1 ? d.D : d.N;     // contraction length (multiple of 4)
  // active-column compaction as in k_simt_probe
  const int space = pflat > 0 ? 0 : t, ncs = pflat > 0 ? pflat : d.P;
  const int nlist = p.b.m_act[space];
  if (j0 >= 4 * nlist) return;                   // CTA-uniform
  const int ngrp = min(SBN / 4, nlist - j0 / 4);
  __shared__ int sgrp[SBN / 4];
  if (tid < SBN / 4) sgrp[tid] = tid < ngrp ? p.b.act[(size_t)space * d.Pp / 4 * (pflat > 0 ? d.Tl : 1) + j0 / 4 + tid] : 0;
  __syncthreads();
  const int ncol = 4 * ngrp;
  const size_t gb = pflat > 0 ? 0 : (size_t)t * d.Pp;
  const size_t fb = pflat > 0 ? 0 : (size_t)t * d.P;
  if (STAGE == 2 && rt == 0 && tid == 0) atomicAdd(p.b.histp + u, SBN);   // columns multiplied
  const float *__restrict__ amat = STAGE == 1 ? p.b.PT + (size_t)t * d.phi_task_stride
                                              : p.phi + (size_t)t * d.phi_task_stride;
  const float *__restrict__ bmat = (STAGE == 1 ? p.b.D32 : p.b.Uh) + gb;
  const size_t ldv = (size_t)d.ldv;
  const uint32_t sa0 = (uint32_t)__cvta_generic_to_shared(ring);
  // a thread's copies: slab rows kr = tid/32 + 4v (v < 4), 4 entries at (tid%32)·4, A and B alike;
  // its source columns and their validity are fixed for the whole K loop
  const int kr0 = tid >> 5, c4 = (tid & 31) * 4;
  const bool oka_m = m0 + c4 < M, okb_c = c4 < ncol;
  const float *asrc = amat + (size_t)kr0 * M + m0 + c4;
  const float *bsrc = bmat + (size_t)kr0 * ldv + (okb_c ? 4 * sgrp[c4 >> 2] : 0);
  const uint32_t st0 = sa0 + 4u * (uint32_t)(kr0 * SLD + c4);
  const char *apn = reinterpret_cast<const char *>(oka_m ? asrc : amat);   // LEAN: the next slab's sources
  const char *bpn = reinterpret_cast<const char *>(okb_c ? bsrc : bmat);
  const size_t a4 = oka_m ? (size_t)16 * M : 0, b4 = okb_c ? (size_t)16 * ldv : 0;   // bytes per 4 k rows
  auto issue = [&](int kt) {
    const int k0 = kt * KBK;
    const uint32_t so = st0 + 4u * (uint32_t)((kt % KST) * 2 * KBK * SLD);
    if (LEAN && k0 + KBK <= KD) {               // a whole slab inside the contraction (CTA-uniform)
      const uint32_t na = oka_m ? 16u : 0u, nb = okb_c ? 16u : 0u;
#pragma unroll
      for (int v = 0; v < KBK / 4; ++v) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(so + 4u * (uint32_t)(4 * v * SLD)),
                     "l"(apn + v * a4), "r"(na) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(so + 4u * (uint32_t)((KBK + 4 * v) * SLD)),
                     "l"(bpn + v * b4), "r"(nb) : "memory");
      }
      apn += (KBK / 4) * a4;
      bpn += (KBK / 4) * b4;
      return;
    }
#pragma unroll
    for (int v = 0; v < KBK / 4; ++v) {
      const bool kin = k0 + kr0 + 4 * v < KD;
      const bool oa = oka_m && kin, ob = okb_c && kin;
      cp_async16(so + 4u * (uint32_t)(4 * v * SLD), oa ? asrc + (size_t)(k0 + 4 * v) * M : amat, oa);
      cp_async16(so + 4u * (uint32_t)((KBK + 4 * v) * SLD), ob ? bsrc + (size_t)(k0 + 4 * v) * ldv : bmat, ob);
    }
  };

  // acc2[ip][j]: rows (2ip, 2ip+1) of this thread's 16 (ip = 2g + i/2: ty·4 + i + 32g), column j of
  // its 8 (tx·4 + (j&3) + 64·(j>>2))
  float2 acc2[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc2[i][j] = make_float2(0.f, 0.f);
#pragma unroll
  for (int q = 0; q < 32; ++q) tot4[q * QTH + tid] = make_float4(0.f, 0.f, 0.f, 0.f);
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
    const float *As = ring + slot * 2 * KBK * SLD + ty * 4, *Bs = ring + (slot * 2 + 1) * KBK * SLD + tx * 4;
    float4 a[4], b[2];
#pragma unroll
    for (int g = 0; g < 4; ++g) a[g] = *reinterpret_cast<const float4 *>(As + 32 * g);
#pragma unroll
    for (int h = 0; h < 2; ++h) b[h] = *reinterpret_cast<const float4 *>(Bs + 64 * h);
#pragma unroll
    for (int kk = 0; kk < KBK; ++kk) {
      float4 na[4], nb[2];
      if (kk + 1 < KBK) {                       // next k's operands before this k's FMAs
#pragma unroll
        for (int g = 0; g < 4; ++g) na[g] = *reinterpret_cast<const float4 *>(As + (kk + 1) * SLD + 32 * g);
#pragma unroll
        for (int h = 0; h < 2; ++h) nb[h] = *reinterpret_cast<const float4 *>(Bs + (kk + 1) * SLD + 64 * h);
      }
      float2 ap[8];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        ap[2 * g] = make_float2(a[g].x, a[g].y);
        ap[2 * g + 1] = make_float2(a[g].z, a[g].w);
      }
      const float bv[8] = {b[0].x, b[0].y, b[0].z, b[0].w, b[1].x, b[1].y, b[1].z, b[1].w};
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc2[i][j] = __ffma2_rn(ap[i], make_float2(bv[j], bv[j]), acc2[i][j]);
      if (kk + 1 < KBK) {
#pragma unroll
        for (int g = 0; g < 4; ++g) a[g] = na[g];
        b[0] = nb[0];
        b[1] = nb[1];
      }
    }
    if ((kt + 1) % FLUSH == 0 || kt + 1 == nk) {   // totals in shared memory (thread-private slots)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float4 tt = tot4[(i * 4 + h) * QTH + tid];
          if (VAR & 4) {                           // packed adds (FADD2): the same round-to-nearest sums
            const float2 lo = __fadd2_rn(make_float2(tt.x, tt.y), acc2[i][2 * h]);
            const float2 hi = __fadd2_rn(make_float2(tt.z, tt.w), acc2[i][2 * h + 1]);
            tt = make_float4(lo.x, lo.y, hi.x, hi.y);
          } else {
            tt.x += acc2[i][2 * h].x;
            tt.y += acc2[i][2 * h].y;
            tt.z += acc2[i][2 * h + 1].x;
            tt.w += acc2[i][2 * h + 1].y;
          }
          tot4[(i * 4 + h) * QTH + tid] = tt;
          acc2[i][2 * h] = acc2[i][2 * h + 1] = make_float2(0.f, 0.f);
        }
    }
  }
  cp_wait<0>();
  // outputs: row m0 + 32g + ty·4 + r (g, r < 4) = tot slot ip = 2g + r/2, .{x|z} (r even) / .{y|w};
  // columns j0 + 64h + tx·4 + q: slot column pair (2h + q/2), element q&1
  if (STAGE == 1) {                             // U [N][ldv]
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + 32 * g + ty * 4 + r;
        if (m >= M) continue;
        const int ip = 2 * g + r / 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = h * 64 + tx * 4;
          if (c >= ncol) continue;
          const float4 t0 = tot4[(ip * 4 + 2 * h) * QTH + tid], t1 = tot4[(ip * 4 + 2 * h + 1) * QTH + tid];
          // slot (ip, hh) = {col 2hh: (row 2ip, row 2ip+1), col 2hh+1: (row 2ip, row 2ip+1)}
          const float4 o = (r & 1) ? make_float4(t0.y, t0.w, t1.y, t1.w) : make_float4(t0.x, t0.z, t1.x, t1.z);
          *reinterpret_cast<float4 *>(p.b.Uh + (size_t)m * ldv + gb + 4 * sgrp[c >> 2]) = o;
        }
      }
  } else {                                      // W = βΦᵀU + α ⊙ d (fp64, one rounding), dᵀW partials
    const double beta = p.beta;
    const int warp = tid >> 5, lane = tid & 31;
    double *sal = reinterpret_cast<double *>(ring);   // α of the tile's rows per cluster (idle ring)
    __syncthreads();
    for (int e = tid; e < d.C * SBM; e += QTH) {
      const int c = e / SBM, r = e % SBM;
      sal[e] = m0 + r < M ? p.b.alpha64[(size_t)c * d.D + m0 + r] : 0.0;
    }
    __syncthreads();
    double dot[8];
    const double *al[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      dot[q] = 0.0;
      const int c = (q >> 2) * 64 + tx * 4 + (q & 3);
      const int jc = min(4 * sgrp[min(c, ncol - 1) >> 2] + (c & 3), ncs - 1);
      al[q] = sal + (size_t)(((fb + jc) % d.P) / d.K) * SBM - m0;
    }
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + 32 * g + ty * 4 + r;
        if (m >= M) continue;
        const int ip = 2 * g + r / 2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = h * 64 + tx * 4;
          if (c >= ncol) continue;
          const float4 t0 = tot4[(ip * 4 + 2 * h) * QTH + tid], t1 = tot4[(ip * 4 + 2 * h + 1) * QTH + tid];
          const float accq[4] = {(r & 1) ? t0.y : t0.x, (r & 1) ? t0.w : t0.z, (r & 1) ? t1.y : t1.x,
                                 (r & 1) ? t1.w : t1.z};
          const size_t o = (size_t)m * ldv + gb + 4 * sgrp[c >> 2];
          const float4 dv = *reinterpret_cast<const float4 *>(p.b.D32 + o);
          const float dq[4] = {dv.x, dv.y, dv.z, dv.w};
          float wq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            wq[q] = (float)fma(beta, (double)accq[q], al[4 * h + q][m] * (double)dq[q]);
            dot[4 * h + q] += (double)dq[q] * (double)wq[q];
          }
          *reinterpret_cast<float4 *>(p.b.W + o) = make_float4(wq[0], wq[1], wq[2], wq[3]);
        }
      }
    // dᵀW over this tile's 128 rows: the ty pair inside a warp, then the 4 warps (fixed order)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double v = dot[q] + __shfl_xor_sync(0xffffffffu, dot[q], 16);
      if (lane < 16) red[warp][(q >> 2) * 64 + tx * 4 + (q & 3)] = v;
    }
    __syncthreads();
    const int jt = tid < ncol ? 4 * sgrp[tid >> 2] + (tid & 3) : ncs;
    if (jt < ncs) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < QTH / 32; ++w) s += red[w][tid];
      p.b.dAd[(fb + jt) * d.nRT2 + rt] = s;
    }
  }
}

// ---- fp64 mean columns ----------------------------------------------------------------------------
__device__ __forceinline__ bool task_mean_active(const KParams &p, int t) {
  int a = 0;
  for (int c = 0; c < p.d.C; ++c) a |= (p.b.flagm[(size_t)t * p.d.C + c] == 1);
  return a != 0;
}

// The mean-column kernels run on a second stream beside the probe SGEMMs (run_simt_cg): 128 threads
// and ≤ 80 registers, so that with the 1-CTA SGEMM form (210 registers × 256 threads) a mean CTA fits
// on an SM next to it and streams Φ from HBM while its FMAs run; with the default 2-CTA form (all
// registers taken) the mean CTAs interleave with the SGEMM CTAs at CTA boundaries.
// Both mean kernels: C[m][c] = Σ_k A[k][m]·B[k][c] in fp64, A the M-major fp32 matrix (stage 1: Φᵀ
// [D][N]; stage 2: Φ [N][D]) in 16-k slabs (a thread per row m: conflict-free reads, no transposes),
// B the C mean columns (stage 1: Dm [C][D] read as [k][c]; stage 2: Um [N][Cp]).  Double-buffered
// shared memory fed from registers: the next slab's loads are issued before this slab's FMAs.
// grid (ceil(M/128), T_loc); stage 2 adds α ⊙ Dm and the dᵀWm partial of its 128 rows.
template <int STAGE>
__global__ void __launch_bounds__(MTH) k_simt_mean(KParams p, int u) {
  __shared__ __align__(16) float As[2][MBK][SBM];
  __shared__ double Bm[2][MBK][MAXC];
  __shared__ double red[MTH / 32][MAXC];
  if (loop_done(p, u)) return;
  const Dims &d = p.d;
  const int t = blockIdx.y + p.toff, tid = threadIdx.x, rt = blockIdx.x, m0 = rt * SBM;
  if (!task_mean_active(p, t)) return;
  const int M = STAGE == 1 ? d.N : d.D, KD = STAGE == 1 ? d.D : d.N, C = d.C;
  const float *__restrict__ amat = (STAGE == 1 ? p.b.PT : p.phi) + (size_t)t * d.phi_task_stride;
  const double *__restrict__ dm = p.b.Dm + (size_t)t * C * d.D;
  const double *__restrict__ um = p.b.Um + (size_t)t * d.N * d.Cp;
  constexpr int NA = MBK * SBM / 4 / MTH;      // float4 of A per thread and slab
  constexpr int NB = MBK * MAXC / MTH;         // B entries per thread and slab (C ≤ MAXC)
  float4 ra[NA];
  double rb[NB];
  auto gload = [&](int k0) {
#pragma unroll
    for (int v = 0; v < NA; ++v) {
      const int idx = tid + v * MTH, kr = idx >> 5, c4 = (idx & 31) * 4, k = k0 + kr;
      ra[v] = (k < KD && m0 + c4 < M) ? ldcs4(amat + (size_t)k * M + m0 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int v = 0; v < NB; ++v) {
      const int e = tid + v * MTH, kk = e / MAXC, c = e % MAXC, k = k0 + kk;
      rb[v] = (c < C && k < KD) ? (STAGE == 1 ? dm[(size_t)c * d.D + k] : um[(size_t)k * d.Cp + c]) : 0.0;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int v = 0; v < NA; ++v) {
      const int idx = tid + v * MTH;
      *reinterpret_cast<float4 *>(&As[buf][idx >> 5][(idx & 31) * 4]) = ra[v];
    }
#pragma unroll
    for (int v = 0; v < NB; ++v) {
      const int e = tid + v * MTH;
      Bm[buf][e / MAXC][e % MAXC] = rb[v];
    }
  };
  double acc[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) acc[c] = 0.0;
  const int nk = (KD + MBK - 1) / MBK;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) gload((kt + 1) * MBK);
#pragma unroll 4
    for (int kk = 0; kk < MBK; ++kk) {
      const double a = (double)As[buf][kk][tid];
      const double2 *bb = reinterpret_cast<const double2 *>(Bm[buf][kk]);
#pragma unroll
      for (int c2 = 0; c2 < MAXC / 2; ++c2) {
        if (2 * c2 >= C) break;
        const double2 bv = bb[c2];              // two clusters per broadcast load
        acc[2 * c2] = fma(a, bv.x, acc[2 * c2]);
        acc[2 * c2 + 1] = fma(a, bv.y, acc[2 * c2 + 1]);
      }
    }
    if (kt + 1 < nk) sstore(buf ^ 1);           // that buffer's readers passed the last barrier
    __syncthreads();
  }
  const int m = m0 + tid;
  if (STAGE == 1) {
    if (m < M) {
#pragma unroll
      for (int c = 0; c < MAXC; ++c)
        if (c < C) p.b.Um[((size_t)t * d.N + m) * d.Cp + c] = acc[c];
    }
    return;
  }
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    if (c >= C) break;
    double v = 0.0;
    if (m < M) {
      const size_t o = ((size_t)t * C + c) * d.D + m;
      const double dv = p.b.Dm[o];
      const double w = fma(p.beta, acc[c], p.b.alpha64[(size_t)c * d.D + m] * dv);
      p.b.Wm[o] = w;
      v = dv * w;
    }
    v = warp_sum_d(v);
    if (lane == 0) red[warp][c] = v;
  }
  __syncthreads();
  if (tid < C) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < MTH / 32; ++w) sum += red[w][tid];
    p.b.dAdm[((size_t)t * C + tid) * d.nRT2 + rt] = sum;
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

// Probe columns, d-major: a CTA updates 32 consecutive columns g = 32·blockIdx.x + lane (one lane per
// column, every global access a 128-byte row segment); its NW warps split the D rows, per-column sums
// are reduced over the warps in fixed order.  Alg. 1 lines 3-7 with fp64 γ_u, ξ_u applied in fp64.
template <int NW>
__device__ void simt_update_probes(const KParams &p, int u) {
  __shared__ double sred[NW][32];
  __shared__ double sgam[32];
  __shared__ int sact[32];
  const Dims &d = p.d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = (blockIdx.x + p.toff * d.Pp / 32) * 32 + lane;   // a task window starts on a 32-column block
  const int t = g / d.Pp, j = g % d.Pp;
  const bool col = t < d.Tl && j < d.P;
  const size_t gi = (size_t)t * d.P + j;     // per-column state index
  const bool active = col && p.b.flag[gi] == 1;
  if (!__syncthreads_or(active)) return;
  // dᵀAd: the nRT2 row-tile partials, split over the warps
  double dp = 0.0;
  if (active)
    for (int i = warp; i < d.nRT2; i += NW) dp += p.b.dAd[gi * d.nRT2 + i];
  sred[warp][lane] = dp;
  __syncthreads();
  if (warp == 0) {
    double dAd = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) dAd += sred[w][lane];
    int act = active;
    if (active) {
      atomicAdd(p.b.hist + u, 1);
      if (atomicMax(p.b.tmark + t, u + 1) < u + 1) atomicAdd(p.b.histt + u, 1);   // tasks active at step u
      if (!(dAd > 0.0)) {  // Alg. 1 line 3 breakdown
        report_simt(p.b.status, ST_BREAKDOWN, d.t0 + t, j, u + 1);
        p.b.flag[gi] = 0;
        act = 0;
      }
    }
    sact[lane] = act;
    sgam[lane] = act ? p.b.rr[gi] / dAd : 0.0;
  }
  __syncthreads();
  const bool go = sact[lane] != 0;
  const double gam = sgam[lane];
  const size_t ldv = (size_t)d.ldv;
  double acc = 0.0;
  if (go) {
    // 4 rows per iteration: 16 independent 128-byte loads in flight per warp
    for (int i0 = warp; i0 < d.D; i0 += 4 * NW) {
      float dv[4], xv[4], wv[4], rv[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = i0 + NW * v;
        if (i < d.D) {
          const size_t o = (size_t)i * ldv + g;
          dv[v] = p.b.D32[o]; xv[v] = p.b.X[o]; wv[v] = p.b.W[o]; rv[v] = p.b.R[o];
        }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = i0 + NW * v;
        if (i < d.D) {
          const size_t o = (size_t)i * ldv + g;
          const float x = (float)fma(gam, (double)dv[v], (double)xv[v]);
          const float r = (float)fma(-gam, (double)wv[v], (double)rv[v]);
          p.b.X[o] = x;
          p.b.R[o] = r;
          acc = fma((double)r, (double)r, acc);
        }
      }
    }
  }
  __syncthreads();                              // sred reuse
  sred[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    double rrn = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) rrn += sred[w][lane];
    double xi = 0.0;
    int cont = 0;
    if (go) {
      const double rr = p.b.rr[gi];
      xi = rrn / rr;
      const bool conv = sqrt(rrn) <= p.tol * sqrt((double)d.D);   // ‖b‖ = ‖p‖ = √D (A5)
      const bool stop = conv || (u + 1 >= d.cap);
      p.b.gam[gi * d.cap + u] = gam;
      p.b.xi[gi * d.cap + u] = xi;
      p.b.steps[gi] = u + 1;
      p.b.rr[gi] = rrn;
      if (stop) p.b.flag[gi] = conv ? 0 : 2;
      else atomicAdd(p.b.alive + u, 1);
      cont = !stop;
    }
    sact[lane] = cont;
    sgam[lane] = xi;
  }
  __syncthreads();
  if (sact[lane]) {
    const double xi = sgam[lane];
    for (int i0 = warp; i0 < d.D; i0 += 4 * NW) {
      float dv[4], rv[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = i0 + NW * v;
        if (i < d.D) {
          const size_t o = (size_t)i * ldv + g;
          dv[v] = p.b.D32[o]; rv[v] = p.b.R[o];
        }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = i0 + NW * v;
        if (i < d.D) p.b.D32[(size_t)i * ldv + g] = (float)fma(xi, (double)dv[v], (double)rv[v]);
      }
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

// blocks [0, nbp): probe column groups (simt_update_probes); then NW mean columns per block (a warp each)
// NW warps per CTA: 8 (default, 256 threads × 80 registers); 4 (CMTCS_SIMT_UPDW=4): 128 threads of
// ≤ 64 registers — exactly what two resident SGEMM CTAs (2 × 128 × 224 registers) leave of an SM, so
// that one task half's update could run beside the other half's SGEMMs (run_simt_cg) — measured
// slower (C4 32 tasks 1227 → 1299 ms per EM iteration: the narrower update itself loses more than
// the overlap gains).
template <int NW>
__global__ void __launch_bounds__(32 * NW, NW == 4 ? 8 : 1) k_simt_update(KParams p, int u, int nbp) {
  if (loop_done(p, u)) return;
  const Dims &d = p.d;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(p.b.u, u + 1);   // CG steps executed (either task half)
  if ((int)blockIdx.x < nbp) {
    simt_update_probes<NW>(p, u);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int w = p.toff * d.C + (blockIdx.x - nbp) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (w >= (p.tcnt ? p.toff + p.tcnt : d.Tl) * d.C) return;
  const int t = w / d.C, c = w % d.C;
  if (p.b.flagm[(size_t)t * d.C + c] != 1) return;
  if (lane == 0) {
    if (atomicMax(p.b.tmark + t, u + 1) < u + 1) atomicAdd(p.b.histt + u, 1);
    atomicAdd(p.b.histm + u, 1);
  }
  simt_update_mean(p, t, c, u, lane);
}

// Active 4-column groups of every column space (a task's P columns, or all tasks' in the flat
// shared-Φ GEMM), in order: act[space·G + i], count m_act[space] (G = Pp/4, or T_loc·P/4 flat).  One
// warp per space, ballot compaction.
__global__ void k_simt_groups(KParams p, int u, int pflat) {
  if (loop_done(p, u)) return;
  const Dims &d = p.d;
  const int space = blockIdx.x + p.toff, lane = threadIdx.x;   // (flat: one space, toff = 0)
  const int ncs = pflat > 0 ? pflat : d.P, ng = (ncs + 3) / 4;
  const size_t fb = pflat > 0 ? 0 : (size_t)space * d.P;
  const size_t lb = (size_t)space * d.Pp / 4 * (pflat > 0 ? d.Tl : 1);
  int cnt = 0;
  for (int q0 = 0; q0 < ng; q0 += 32) {
    const int q = q0 + lane;
    bool a = false;
    if (q < ng)
#pragma unroll
      for (int e = 0; e < 4; ++e) a |= (4 * q + e < ncs) && p.b.flag[fb + 4 * q + e] == 1;
    const unsigned m = __ballot_sync(0xffffffffu, a);
    if (a) p.b.act[lb + cnt + __popc(m & ((1u << lane) - 1u))] = q;
    cnt += __popc(m);
  }
  if (lane == 0) p.b.m_act[space] = cnt;
}

}  // namespace

// The CG loop of an E-step on the CUDA cores.  Termination is checked on the host every
// SimtTiming::B steps (alive[u] read back through pinned memory); the kernels of steps past the last
// one return at once.  *launches counts the kernels launched; with `tm` the operator (stage 1 → the
// end of stage 2, mean kernels included) and update durations are accumulated from CUDA events.
cudaError_t run_simt_cg(const KParams &p, int *h_alive, int64_t *launches, SimtTiming *tm, const SimtStreams &ss,
                        cudaStream_t s) {
  const Dims &d = p.d;
  const int pflat = d.shared_phi && d.P % 4 == 0 ? d.Tl * d.P : 0;   // Pp == P: U rows contiguous too
  const int gx = ((pflat ? pflat : d.P) + SBN - 1) / SBN, gz = pflat ? 1 : d.Tl;
  const dim3 g1(gx, (d.N + SBM - 1) / SBM, gz);
  const dim3 g2(gx, (d.D + SBM - 1) / SBM, gz);
  const dim3 gm1((d.N + SBM - 1) / SBM, d.Tl), gm2((d.D + SBM - 1) / SBM, d.Tl);
  static const int updw = getenv("CMTCS_SIMT_UPDW") && atoi(getenv("CMTCS_SIMT_UPDW")) == 4 ? 4 : 8;   // warps per update CTA
  const int nbp = (d.ldv + 31) / 32, gu = nbp + (d.Tl * d.C + updw - 1) / updw;
  constexpr int B = SimtTiming::B;
  cudaError_t e = cudaSuccess;
  // form: 0 the 4-warp 16 × 8-per-thread SGEMM (default); CMTCS_SIMT_FORM=1 the 8-warp 8 × 8 form with 2
  // CTAs per SM, 2 the same with 1 CTA per SM (C4, 32 tasks: 1387 vs 1426 ms per EM iteration)
  static const int form = getenv("CMTCS_SIMT_FORM") ? atoi(getenv("CMTCS_SIMT_FORM")) : 0;
  const bool smt = form != 2;
  static const int var = getenv("CMTCS_SIMT_VAR") ? atoi(getenv("CMTCS_SIMT_VAR")) & 15 : 3;
  static bool configured = false;   // dynamic shared memory above 48 KB (one process per GPU)
  if (!configured) {
    const int s0 = (int)PCfg<false>::SMEM, s1 = (int)PCfg<true>::SMEM;
    e = cudaFuncSetAttribute(k_simt_probe<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s0);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s0);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1);
#define CMTCS_P4_ATTR(V)                                                                                       \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe4<1, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QSMEM); \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_simt_probe4<2, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QSMEM);
    CMTCS_P4_ATTR(0) CMTCS_P4_ATTR(1) CMTCS_P4_ATTR(2) CMTCS_P4_ATTR(3) CMTCS_P4_ATTR(4) CMTCS_P4_ATTR(5) CMTCS_P4_ATTR(6) CMTCS_P4_ATTR(7) CMTCS_P4_ATTR(11) CMTCS_P4_ATTR(14)
#undef CMTCS_P4_ATTR
    if (e != cudaSuccess) return e;
    configured = true;
  }
  e = cudaMemsetAsync(p.b.u, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  // Two task halves as two independent CG loops (default where every task has its own Φ and the second
  // half starts on a 32-column block and a half fills the GPU; CMTCS_SIMT_SPLIT=0: one loop, 2: split
  // whatever the size): half 0 on `s`, half 1 on the side
  // stream, each with its own alive[] array.  A column's arithmetic is unchanged (same kernels, same
  // tiles); what changes is what shares the GPU: one half's HBM-bound update and mean kernels and the
  // partial last wave of its SGEMMs run beside the other half's FMA-bound SGEMMs.  Per-step event
  // timing (op_ms / upd_ms) does not apply to overlapped phases and stays 0.
  static const int split = getenv("CMTCS_SIMT_SPLIT") ? atoi(getenv("CMTCS_SIMT_SPLIT")) : 1;
  int th = 0;
  if (split && form == 0 && !pflat && d.Tl >= 2) {
    int align = 32, a = d.Pp % 32;
    while (a) { const int r = align % a; align = a; a = r; }   // gcd(32, Pp) (Pp % 32 == 0: 32)
    align = 32 / align;                                        // tasks per whole 32-column block
    th = d.Tl / 2 / align * align;
    // auto (1): only where a half's stage-1 SGEMM has a CTA for every SM — below that the loop is
    // launch-latency bound and the longer in-stream chain loses (C2: 25.4 → 20.9 EM it/s); 2: always
    if (split == 1 && (long long)gx * g1.y * th < 148) th = 0;
  }
  if (th > 0) {
    KParams ph[2] = {p, p};
    ph[0].toff = 0, ph[0].tcnt = th;
    ph[1].toff = th, ph[1].tcnt = d.Tl - th;
    ph[1].b.alive = p.b.alive + d.cap;
    const cudaStream_t st[2] = {s, ss.side};
    e = cudaEventRecord(ss.fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ss.side, ss.fork, 0);
    if (e != cudaSuccess) return e;
    for (int u = 0; u < d.cap; ++u) {
      for (int h = 0; h < 2; ++h) {
        const KParams &q = ph[h];
        const dim3 h1(gx, g1.y, q.tcnt), h2(gx, g2.y, q.tcnt), hm1(gm1.x, q.tcnt), hm2(gm2.x, q.tcnt);
        const int hbp = (q.tcnt * d.Pp + 31) / 32, hu = hbp + (q.tcnt * d.C + updw - 1) / updw;
        k_simt_groups<<<q.tcnt, 32, 0, st[h]>>>(q, u, 0);
        k_simt_mean<1><<<hm1, MTH, 0, st[h]>>>(q, u);
        k_simt_mean<2><<<hm2, MTH, 0, st[h]>>>(q, u);
        switch (var) {
#define CMTCS_P4_RUN(V)                                             \
  case V:                                                           \
    k_simt_probe4<1, V><<<h1, QTH, QSMEM, st[h]>>>(q, u, 0);        \
    k_simt_probe4<2, V><<<h2, QTH, QSMEM, st[h]>>>(q, u, 0);        \
    break;
          CMTCS_P4_RUN(1) CMTCS_P4_RUN(2) CMTCS_P4_RUN(3) CMTCS_P4_RUN(4) CMTCS_P4_RUN(5) CMTCS_P4_RUN(6) CMTCS_P4_RUN(7) CMTCS_P4_RUN(11) CMTCS_P4_RUN(14)
          default: CMTCS_P4_RUN(0)
#undef CMTCS_P4_RUN
        }
        if (updw == 8) k_simt_update<8><<<hu, 256, 0, st[h]>>>(q, u, hbp);
        else k_simt_update<4><<<hu, 128, 0, st[h]>>>(q, u, hbp);
      }
      *launches += 12;
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      if (u % B == B - 1 || u + 1 == d.cap) {
        for (int h = 0; h < 2 && e == cudaSuccess; ++h)
          e = cudaMemcpyAsync(h_alive + h, ph[h].b.alive + u, sizeof(int), cudaMemcpyDeviceToHost, st[h]);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ss.side);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        if (h_alive[0] == 0 && h_alive[1] == 0) break;
      }
    }
    e = cudaEventRecord(ss.join, ss.side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ss.join, 0);
    return e;
  }
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
    k_simt_groups<<<pflat ? 1 : d.Tl, 32, 0, s>>>(p, u, pflat);
    // fork: the mean columns (fp64, HBM-bound) on the side stream, the probe SGEMMs (FMA-bound) here
    cudaEventRecord(ss.fork, s);
    cudaStreamWaitEvent(ss.side, ss.fork, 0);
    k_simt_mean<1><<<gm1, MTH, 0, ss.side>>>(p, u);
    k_simt_mean<2><<<gm2, MTH, 0, ss.side>>>(p, u);
    cudaEventRecord(ss.join, ss.side);
    if (form == 0) {
      switch (var) {
#define CMTCS_P4_RUN(V)                                        \
  case V:                                                      \
    k_simt_probe4<1, V><<<g1, QTH, QSMEM, s>>>(p, u, pflat);   \
    k_simt_probe4<2, V><<<g2, QTH, QSMEM, s>>>(p, u, pflat);   \
    break;
        CMTCS_P4_RUN(1) CMTCS_P4_RUN(2) CMTCS_P4_RUN(3) CMTCS_P4_RUN(4) CMTCS_P4_RUN(5) CMTCS_P4_RUN(6) CMTCS_P4_RUN(7) CMTCS_P4_RUN(11) CMTCS_P4_RUN(14)
        default: CMTCS_P4_RUN(0)
#undef CMTCS_P4_RUN
      }
    } else if (smt) {
      k_simt_probe<1, true><<<g1, STH, PCfg<true>::SMEM, s>>>(p, u, pflat);
      k_simt_probe<2, true><<<g2, STH, PCfg<true>::SMEM, s>>>(p, u, pflat);
    } else {
      k_simt_probe<1, false><<<g1, STH, PCfg<false>::SMEM, s>>>(p, u, pflat);
      k_simt_probe<2, false><<<g2, STH, PCfg<false>::SMEM, s>>>(p, u, pflat);
    }
    cudaStreamWaitEvent(s, ss.join, 0);
    if (tm) cudaEventRecord(tm->ev[3 * slot + 1], s);
    if (updw == 8) k_simt_update<8><<<gu, 256, 0, s>>>(p, u, nbp);
    else k_simt_update<4><<<gu, 128, 0, s>>>(p, u, nbp);
    if (tm) cudaEventRecord(tm->ev[3 * slot + 2], s);
    *launches += 6;
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
