// K1 — the batched normal operator W = βΦ_tᵀ(Φ_t V) + α_{c(m)} ⊙ V over every active CG column
// of every task ("A := βΦᵀΦ + diag(α)", "solve all TC(K+1) systems
// simultaneously ... A never needs to be explicitly computed").
//
// Two contractions per CG step (never forming ΦᵀΦ, N = D/4 makes this the cheaper order):
//   stage 1  U[t][n][j] = Σ_d Φ_t[n][d] · V[t][act_j][d]          (rows n,  K = D)
//   stage 2  W[t][act_j][d] = β Σ_n Φ_t[n][d] · U[t][n][j] + α ⊙ V (rows d,  K = N)
//            + the per-row-tile partial dᵀ(Ad) of Alg. 1 line 3, accumulated in fp64.
// Probe columns are fp32 (FFMA, register-blocked 8x4 per thread, 128x64 CTA tile, smem double
// buffer); converged columns are compacted away (act list), so retired columns cost nothing.
// The C mean columns of a task run as one extra fp64 CTA per row tile (blockIdx.x == nCT) that
// reads the same Φ tile (DFMA), keeping μ in fp64 end to end.
#include "cmtcs_internal.cuh"

namespace cmtcs {

namespace {

constexpr int BR = OP_BR, BC = OP_BC, BK = OP_BK;
constexpr int ALD = BR + 4;   // padded leading dims (keep 16-byte alignment for LDS.128)
constexpr int BLD = BC + 4;

struct __align__(16) OpSmem {
  float A[2][BK][ALD];
  union {
    float B[2][BK][BLD];
    double Bm[2][BK][MAXC];
  };
  double red[16][BC];          // stage-2 dot partials (probe tile)
  int m;
  int mc;
};

__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }

// Builds the compacted list of active probe columns of task t (ascending) in s_act; returns count.
__device__ int build_act(const int *flag, int P, int *s_act, int *s_m) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    int cnt = 0;
    for (int base = 0; base < P; base += 32) {
      const int j = base + tid;
      const int f = (j < P) ? flag[j] : 0;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (f) s_act[cnt + __popc(bal & ((1u << tid) - 1u))] = j;
      cnt += __popc(bal);
    }
    if (tid == 0) *s_m = cnt;
  }
  __syncthreads();
  return *s_m;
}

// ---------------------------------------------------------------------------------------------
// stage 1
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(OP_THREADS) k_stage1(KParams p, int u, const double *__restrict__ mu_src,
                                                       int mu_only) {
  extern __shared__ int s_act[];
  __shared__ OpSmem sm;
  const Dims &d = p.d;
  const int t = blockIdx.z, rt = blockIdx.y, ct = blockIdx.x, tid = threadIdx.x;
  const int N = d.N, D = d.D, P = d.P, C = d.C;
  const float *__restrict__ phi = p.phi + (size_t)t * d.phi_task_stride;
  const int n0 = rt * BR;
  const int nk = (D + BK - 1) / BK;

  // A-tile loader: Φ[n0 + r][k0 + 4q .. +3] → A[k][r] (transposed; 2 float4 per thread)
  auto loadA = [&](int k0, float4 *ra) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * OP_THREADS, r = idx >> 2, q = idx & 3;
      const int n = n0 + r, k = k0 + 4 * q;
      ra[i] = (n < N && k < D) ? ld4(phi + (size_t)n * D + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto storeA = [&](int buf, const float4 *ra) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * OP_THREADS, r = idx >> 2, q = idx & 3;
      sm.A[buf][4 * q + 0][r] = ra[i].x;
      sm.A[buf][4 * q + 1][r] = ra[i].y;
      sm.A[buf][4 * q + 2][r] = ra[i].z;
      sm.A[buf][4 * q + 3][r] = ra[i].w;
    }
  };

  if (ct == d.nCT) {
    // ---------------- fp64 mean-column tile: Um[t][n][c] = Σ_d Φ[n][d] μsrc[t][c][d] ----------
    if (!mu_only) {
      int any = 0;
      for (int c = 0; c < C; ++c) any |= p.b.flagm[t * C + c];
      if (!any) return;
    }
    const double *src = mu_src + (size_t)t * C * D;
    const int r = tid & (BR - 1), h = tid >> 7;
    double acc[MAXC / 2];
#pragma unroll
    for (int i = 0; i < MAXC / 2; ++i) acc[i] = 0.0;
    float4 ra[2];
    double rb = 0.0;
    auto loadB = [&](int k0) {
      rb = 0.0;
      if (tid < BK * C) {
        const int c = tid / BK, kk = tid % BK;
        if (k0 + kk < D) rb = src[(size_t)c * D + k0 + kk];
      }
    };
    auto storeB = [&](int buf) {
      if (tid < BK * C) sm.Bm[buf][tid % BK][tid / BK] = rb;
    };
    loadA(0, ra);
    loadB(0);
    storeA(0, ra);
    storeB(0);
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
      const int buf = kc & 1;
      if (kc + 1 < nk) {
        loadA((kc + 1) * BK, ra);
        loadB((kc + 1) * BK);
      }
#pragma unroll 4
      for (int kk = 0; kk < BK; ++kk) {
        const double a = (double)sm.A[buf][kk][r];
#pragma unroll
        for (int i = 0; i < MAXC / 2; ++i)
          if (h + 2 * i < C) acc[i] = fma(a, sm.Bm[buf][kk][h + 2 * i], acc[i]);
      }
      if (kc + 1 < nk) {
        storeA(buf ^ 1, ra);
        storeB(buf ^ 1);
      }
      __syncthreads();
    }
    const int n = n0 + r;
    if (n < N) {
#pragma unroll
      for (int i = 0; i < MAXC / 2; ++i)
        if (h + 2 * i < C) p.b.Um[((size_t)t * N + n) * C + h + 2 * i] = acc[i];
    }
    return;
  }
  if (mu_only) return;

  // ---------------- fp32 probe tile -------------------------------------------------------
  const int m = build_act(p.b.flag + (size_t)t * P, P, s_act, &sm.m);
  if (ct == 0 && rt == 0) {
    // task bookkeeping for this CG step: publish act list, step histograms
    for (int j = tid; j < m; j += OP_THREADS) p.b.act[(size_t)t * P + j] = s_act[j];
    if (tid == 0) {
      p.b.m_act[t] = m;
      int mc = 0;
      for (int c = 0; c < C; ++c) mc += p.b.flagm[t * C + c];
      if (m) atomicAdd(p.b.hist + u, m);
      if (mc) atomicAdd(p.b.histm + u, mc);
      if (m + mc) atomicAdd(p.b.histt + u, 1);
    }
  }
  const int j0 = ct * BC;
  if (j0 >= m) return;

  const int ty = tid >> 4, tx = tid & 15;
  const int cb = tid >> 2, qb = tid & 3;
  const float *bcol = (j0 + cb < m) ? p.b.Dv + ((size_t)t * P + s_act[j0 + cb]) * D : nullptr;
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  float4 ra[2], rb;
  auto loadB = [&](int k0) {
    const int k = k0 + 4 * qb;
    rb = (bcol && k < D) ? ld4(bcol + k) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto storeB = [&](int buf) {
    sm.B[buf][4 * qb + 0][cb] = rb.x;
    sm.B[buf][4 * qb + 1][cb] = rb.y;
    sm.B[buf][4 * qb + 2][cb] = rb.z;
    sm.B[buf][4 * qb + 3][cb] = rb.w;
  };
  loadA(0, ra);
  loadB(0);
  storeA(0, ra);
  storeB(0);
  __syncthreads();
  for (int kc = 0; kc < nk; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nk) {
      loadA((kc + 1) * BK, ra);
      loadB((kc + 1) * BK);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4 *>(&sm.A[buf][kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4 *>(&sm.A[buf][kk][ty * 8 + 4]);
      const float4 bv = *reinterpret_cast<const float4 *>(&sm.B[buf][kk][tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (kc + 1 < nk) {
      storeA(buf ^ 1, ra);
      storeB(buf ^ 1);
    }
    __syncthreads();
  }
  const int jc = j0 + tx * 4;
  if (jc < d.Pp) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int n = n0 + ty * 8 + i;
      if (n < N)
        *reinterpret_cast<float4 *>(p.b.U + ((size_t)t * N + n) * d.Pp + jc) =
            make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// stage 2
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(OP_THREADS) k_stage2(KParams p, int u) {
  __shared__ OpSmem sm;
  const Dims &d = p.d;
  const int t = blockIdx.z, rt = blockIdx.y, ct = blockIdx.x, tid = threadIdx.x;
  const int N = d.N, D = d.D, P = d.P, C = d.C;
  const float *__restrict__ phi = p.phi + (size_t)t * d.phi_task_stride;
  const int d0 = rt * BR;
  const int nk = (N + BK - 1) / BK;
  const double beta = p.beta;

  // A-tile loader: Φ[k0 + kk][d0 + 4q .. +3] → A[kk][4q..] (direct, 2 float4 per thread)
  auto loadA = [&](int k0, float4 *ra) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * OP_THREADS, kk = idx >> 5, q = idx & 31;
      const int n = k0 + kk, dd = d0 + 4 * q;
      ra[i] = (n < N && dd < D) ? ld4(phi + (size_t)n * D + dd) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto storeA = [&](int buf, const float4 *ra) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * OP_THREADS, kk = idx >> 5, q = idx & 31;
      *reinterpret_cast<float4 *>(&sm.A[buf][kk][4 * q]) = ra[i];
    }
  };

  if (ct == d.nCT) {
    // ---------------- fp64 mean-column tile ---------------------------------------------------
    int any = 0;
    for (int c = 0; c < C; ++c) any |= p.b.flagm[t * C + c];
    if (!any) return;
    const int r = tid & (BR - 1), h = tid >> 7;
    double acc[MAXC / 2];
#pragma unroll
    for (int i = 0; i < MAXC / 2; ++i) acc[i] = 0.0;
    float4 ra[2];
    double rb = 0.0;
    const double *um = p.b.Um + (size_t)t * N * C;
    auto loadB = [&](int k0) {
      rb = 0.0;
      if (tid < BK * C) {
        const int kk = tid / C, c = tid % C;
        if (k0 + kk < N) rb = um[(size_t)(k0 + kk) * C + c];
      }
    };
    auto storeB = [&](int buf) {
      if (tid < BK * C) sm.Bm[buf][tid / C][tid % C] = rb;
    };
    loadA(0, ra);
    loadB(0);
    storeA(0, ra);
    storeB(0);
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
      const int buf = kc & 1;
      if (kc + 1 < nk) {
        loadA((kc + 1) * BK, ra);
        loadB((kc + 1) * BK);
      }
#pragma unroll 4
      for (int kk = 0; kk < BK; ++kk) {
        const double a = (double)sm.A[buf][kk][r];
#pragma unroll
        for (int i = 0; i < MAXC / 2; ++i)
          if (h + 2 * i < C) acc[i] = fma(a, sm.Bm[buf][kk][h + 2 * i], acc[i]);
      }
      if (kc + 1 < nk) {
        storeA(buf ^ 1, ra);
        storeB(buf ^ 1);
      }
      __syncthreads();
    }
    // epilogue: Wm = β acc + α ⊙ dm ; partial dᵀW over this row tile
    const int dd = d0 + r;
    double dot[MAXC / 2];
#pragma unroll
    for (int i = 0; i < MAXC / 2; ++i) {
      dot[i] = 0.0;
      const int c = h + 2 * i;
      if (c < C && dd < D) {
        const size_t o = ((size_t)t * C + c) * D + dd;
        const double dv = p.b.Dm[o];
        const double w = fma(beta, acc[i], p.b.alpha64[(size_t)c * D + dd] * dv);
        p.b.Wm[o] = w;
        dot[i] = dv * w;
      }
    }
    // reduce over the 128 rows of each half: warp shuffle, then 4 warps via smem
    double *red = &sm.red[0][0];  // [2 halves][4 warps][MAXC/2]
    const int lane = tid & 31, wq = (tid >> 5) & 3;
#pragma unroll
    for (int i = 0; i < MAXC / 2; ++i) {
      double v = dot[i];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[(h * 4 + wq) * (MAXC / 2) + i] = v;
    }
    __syncthreads();
    if (tid < MAXC) {
      const int hh = tid & 1, i = tid >> 1, c = hh + 2 * i;
      if (c < C) {
        double v = 0.0;
        for (int w = 0; w < 4; ++w) v += red[(hh * 4 + w) * (MAXC / 2) + i];
        p.b.dAdm[((size_t)t * C + c) * d.nRT2 + rt] = v;
      }
    }
    return;
  }

  // ---------------- fp32 probe tile -------------------------------------------------------
  const int m = p.b.m_act[t];
  const int j0 = ct * BC;
  if (j0 >= m) return;
  const int ty = tid >> 4, tx = tid & 15;
  const float *__restrict__ U = p.b.U + (size_t)t * N * d.Pp;
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  float4 ra[2], rb;
  const int kb = tid >> 4, qb = tid & 15;
  auto loadB = [&](int k0) {
    const int n = k0 + kb, j = j0 + 4 * qb;
    rb = (n < N && j < d.Pp) ? ld4(U + (size_t)n * d.Pp + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto storeB = [&](int buf) { *reinterpret_cast<float4 *>(&sm.B[buf][kb][4 * qb]) = rb; };
  loadA(0, ra);
  loadB(0);
  storeA(0, ra);
  storeB(0);
  __syncthreads();
  for (int kc = 0; kc < nk; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nk) {
      loadA((kc + 1) * BK, ra);
      loadB((kc + 1) * BK);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4 *>(&sm.A[buf][kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4 *>(&sm.A[buf][kk][ty * 8 + 4]);
      const float4 bv = *reinterpret_cast<const float4 *>(&sm.B[buf][kk][tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (kc + 1 < nk) {
      storeA(buf ^ 1, ra);
      storeB(buf ^ 1);
    }
    __syncthreads();
  }
  // epilogue: W = β acc + α_c ⊙ d, partial dᵀW (fp64) per column over this row tile
  const float betaf = (float)beta;
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    const int j = j0 + tx * 4 + jj;
    double dot = 0.0;
    if (j < m) {
      const int col = p.b.act[(size_t)t * P + j];
      const int c = col / d.K;
      const size_t base = ((size_t)t * P + col) * D;
      const float *al = p.b.alpha32 + (size_t)c * D;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int dd = d0 + ty * 8 + 4 * h;
        if (dd < D) {
          const float4 dv = ld4(p.b.Dv + base + dd);
          const float4 a4 = ld4(al + dd);
          float4 w;
          w.x = fmaf(betaf, acc[4 * h + 0][jj], a4.x * dv.x);
          w.y = fmaf(betaf, acc[4 * h + 1][jj], a4.y * dv.y);
          w.z = fmaf(betaf, acc[4 * h + 2][jj], a4.z * dv.z);
          w.w = fmaf(betaf, acc[4 * h + 3][jj], a4.w * dv.w);
          *reinterpret_cast<float4 *>(p.b.W + base + dd) = w;
          dot += (double)dv.x * w.x + (double)dv.y * w.y + (double)dv.z * w.z + (double)dv.w * w.w;
        }
      }
    }
    sm.red[ty][tx * 4 + jj] = dot;
  }
  __syncthreads();
  if (tid < BC) {
    const int j = j0 + tid;
    if (j < m) {
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) v += sm.red[i][tid];
      const int col = p.b.act[(size_t)t * P + j];
      p.b.dAd[((size_t)t * P + col) * d.nRT2 + rt] = v;
    }
  }
}

}  // namespace

cudaError_t launch_stage1(const KParams &p, int u, const double *mu_src, bool mu_only, cudaStream_t s) {
  dim3 grid(p.d.nCT + 1, p.d.nRT1, p.d.Tl);
  k_stage1<<<grid, OP_THREADS, sizeof(int) * p.d.P, s>>>(p, u, mu_src ? mu_src : p.b.Dm, mu_only ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_stage2(const KParams &p, int u, cudaStream_t s) {
  dim3 grid(p.d.nCT + 1, p.d.nRT2, p.d.Tl);
  k_stage2<<<grid, OP_THREADS, 0, s>>>(p, u);
  return cudaGetLastError();
}

}  // namespace cmtcs
