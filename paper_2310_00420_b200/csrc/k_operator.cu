// K1 — the batched normal operator W = βΦ_tᵀ(Φ_t V) + α_{c(m)} ⊙ V over every active CG column
// of every task ("A := βΦᵀΦ + diag(α)", "solve all TC(K+1) systems
// simultaneously ... A never needs to be explicitly computed").
//
// Two contractions per CG step (ΦᵀΦ is never formed; N = D/4 makes this the cheaper order):
//   stage 1  U[t][n][j] = Σ_s Σ_{d ∈ slice s} Φ_t[n][d] · V[t][act_j][d]   (rows n, K = D)
//            split-K over S1 slices when T·N is small; the S1 CTAs of a tile form a thread-block
//            cluster and reduce their partial tiles over DSMEM in fixed order (deterministic)
//   stage 2  W[t][act_j][d] = β Σ_n Φ_t[n][d] · U[t][n][j] + α ⊙ V          (rows d, K = N)
//            + the per-row-tile partial dᵀ(Ad) of Alg. 1 line 3, accumulated in fp64.
// Probe columns (fp32): CTA = 8 warps = 128 rows × 96 columns; each warp owns 12 columns and all
// 128 rows (lane: 4 rows × 12 columns, 48 FFMA per k per 4 smem loads).  Converged columns are
// compacted away (act list) and a warp whose 12 columns are all retired skips its FFMAs, so the
// waste is < 12 columns per task.  Φ tiles stream through a 3-stage cp.async ring.
// The C mean columns of a task run as one extra fp64 CTA per row tile (blockIdx.x == nCT) on the
// same Φ tiles (DFMA), keeping μ in fp64 end to end.
#include <cooperative_groups.h>

#include "cmtcs_internal.cuh"

namespace cg = cooperative_groups;

namespace cmtcs {

namespace {

constexpr int BR = OP_BR;       // 128 rows per CTA
constexpr int BC = OP_BC;       // 96 probe columns per CTA
constexpr int BK = OP_BK;       // 16: contraction chunk
constexpr int WC = BC / 8;      // 12 columns per warp
constexpr int ST = 3;           // pipeline stages
constexpr int A1LD = BK + 4;    // stage-1 A tile [r][k]  (row stride 20 floats: conflict-free LDS.128)
constexpr int A2LD = BR + 4;    // stage-2 A tile [k][r]
constexpr int BLD = BC + 4;     // B tile [k][c]

struct __align__(16) Smem1 {
  float A[ST][BR][A1LD];        // 30720 B
  union {
    float B[ST][BK][BLD];       // 19200 B
    double Bm[ST][BK][MAXC];    //  6144 B
  };
  int m;
};

struct __align__(16) Smem2 {
  float A[ST][BK][A2LD];        // 25344 B
  union {
    float B[ST][BK][BLD];
    double Bm[ST][BK][MAXC];
  };
  double red[2][4][MAXC / 2];
};

__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;  // src-size 0 ⇒ zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Compacted list of active probe columns of task t (ascending) in s_act; returns the count.
__device__ int build_act(const int *flag, int P, int *s_act, int *s_m) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    int cnt = 0;
    for (int base = 0; base < P; base += 32) {
      const int j = base + tid;
      const int f = (j < P) ? (flag[j] == 1) : 0;
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
// stage 1:  grid (nCT + 1, nRT1 * S1, Tl)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(OP_THREADS, 2) k_stage1(KParams p, const double *__restrict__ mu_src,
                                                          int mu_only) {
  extern __shared__ __align__(16) unsigned char dsm1[];
  Smem1 &sm = *reinterpret_cast<Smem1 *>(dsm1);
  int *s_act = reinterpret_cast<int *>(dsm1 + sizeof(Smem1));
  const Dims &d = p.d;
  const int t = blockIdx.z, ct = blockIdx.x, tid = threadIdx.x;
  const int rt = blockIdx.y / d.S1, sp = blockIdx.y % d.S1;
  const int N = d.N, D = d.D, P = d.P, C = d.C;
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

  if (ct == d.nCT) {
    // ---------------- fp64 mean-column tile: Um_s[t][n][c] = Σ_{d∈s} Φ[n][d] μsrc[t][c][d] ------
    if (!mu_only) {
      int any = 0;
      for (int c = 0; c < C; ++c) any |= (p.b.flagm[t * C + c] == 1);
      if (!any) return;
      if (tid == 0) atomicMax(p.b.ts + 4 * (*p.b.u), ~globaltimer());
    }
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
      if (n0 + rr < N) p.b.Um[((size_t)t * N + n0 + rr) * C + c] = v;
    }
    if (d.S1 > 1) cl.sync();
    return;
  }
  if (mu_only) return;

  // ---------------- fp32 probe tile -------------------------------------------------------
  const int u = *p.b.u;
  if (tid == 0) atomicMax(p.b.ts + 4 * u, ~globaltimer());  // ~t: max ⇔ min
  const int m = build_act(p.b.flag + (size_t)t * P, P, s_act, &sm.m);
  if (ct == 0 && blockIdx.y == 0) {
    // task bookkeeping for this CG step: publish the act list and the step histograms
    for (int j = tid; j < m; j += OP_THREADS) p.b.act[(size_t)t * P + j] = s_act[j];
    if (tid == 0) {
      p.b.m_act[t] = m;
      int mc = 0;
      for (int c = 0; c < C; ++c) mc += (p.b.flagm[t * C + c] == 1);
      if (m) atomicAdd(p.b.hist + u, m);
      if (mc) atomicAdd(p.b.histm + u, mc);
      if (m + mc) atomicAdd(p.b.histt + u, 1);
    }
  }
  const int j0 = ct * BC;
  if (j0 >= m) return;
  const int w = tid >> 5, l = tid & 31;
  const bool wact = j0 + w * WC < m;   // this warp has at least one active column

  // B tile (register-staged transpose): V[act[j0 + c]][k0 + 4q .. +3] → B[4q + i][c]
  // 384 float4 per stage: idx = tid (+256): c = idx >> 2, q = idx & 3
  const float *bsrc[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int idx = tid + i * OP_THREADS, c = idx >> 2;
    bsrc[i] = (idx < BC * 4 && j0 + c < m) ? p.b.Dv + ((size_t)t * P + s_act[j0 + c]) * D : nullptr;
  }
  float4 rb[2];
  auto loadB = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * OP_THREADS, q = idx & 3;
      const int k = k0 + 4 * q;
      rb[i] = (bsrc[i] && k < ke) ? ld4(bsrc[i] + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto storeB = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * OP_THREADS, c = idx >> 2, q = idx & 3;
      if (idx < BC * 4) {
        sm.B[buf][4 * q + 0][c] = rb[i].x;
        sm.B[buf][4 * q + 1][c] = rb[i].y;
        sm.B[buf][4 * q + 2][c] = rb[i].z;
        sm.B[buf][4 * q + 3][c] = rb[i].w;
      }
    }
  };

  float acc[4][WC];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < WC; ++c) acc[i][c] = 0.f;

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nk) { loadA(s, kb + s * BK); loadB(kb + s * BK); storeB(s); }
    cp_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_wait<ST - 2>();
    __syncthreads();
    const int nx = kc + ST - 1;
    if (nx < nk) { loadA(nx % ST, kb + nx * BK); loadB(kb + nx * BK); }
    cp_commit();
    const int buf = kc % ST;
    if (wact) {
#pragma unroll
      for (int kq = 0; kq < BK / 4; ++kq) {
        float4 a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const float4 *>(&sm.A[buf][l + 32 * i][4 * kq]);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float *brow = &sm.B[buf][4 * kq + kk][w * WC];
          const float4 b0 = *reinterpret_cast<const float4 *>(brow);
          const float4 b1 = *reinterpret_cast<const float4 *>(brow + 4);
          const float4 b2 = *reinterpret_cast<const float4 *>(brow + 8);
          const float b[WC] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float av = kk == 0 ? a[i].x : kk == 1 ? a[i].y : kk == 2 ? a[i].z : a[i].w;
#pragma unroll
            for (int c = 0; c < WC; ++c) acc[i][c] = fmaf(av, b[c], acc[i][c]);
          }
        }
      }
    }
    if (nx < nk) storeB(nx % ST);
  }
  cp_wait<0>();
  const int jc = j0 + w * WC;
  if (d.S1 == 1) {
    if (wact) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int n = n0 + l + 32 * i;
        if (n < N) {
          float *dst = p.b.U + ((size_t)t * N + n) * d.Pp + jc;
#pragma unroll
          for (int q = 0; q < WC / 4; ++q)
            if (jc + 4 * q < d.Pp)
              *reinterpret_cast<float4 *>(dst + 4 * q) =
                  make_float4(acc[i][4 * q], acc[i][4 * q + 1], acc[i][4 * q + 2], acc[i][4 * q + 3]);
        }
      }
    }
    return;
  }
  // split-K: partial tile [BR][BC] in smem (aliases the pipeline buffers), cluster-wide reduction
  __syncthreads();
  float *part = reinterpret_cast<float *>(dsm1);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < WC / 4; ++q)
      *reinterpret_cast<float4 *>(part + (l + 32 * i) * BC + w * WC + 4 * q) =
          wact ? make_float4(acc[i][4 * q], acc[i][4 * q + 1], acc[i][4 * q + 2], acc[i][4 * q + 3])
               : make_float4(0.f, 0.f, 0.f, 0.f);
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  {
    // this CTA (cluster rank sp) owns rows [sp·BR/S1, (sp+1)·BR/S1) of the tile
    const int rows = BR / d.S1, rb = sp * rows;
    const int ncol4 = min(BC, ((m - j0) + 3) & ~3) / 4;   // float4 groups holding active columns
    for (int e = tid; e < rows * ncol4; e += OP_THREADS) {
      const int rr = rb + e / ncol4, q = e % ncol4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int src = 0; src < d.S1; ++src) {   // fixed order: deterministic sum
        const float4 x = *reinterpret_cast<const float4 *>(cl.map_shared_rank(part, src) + rr * BC + 4 * q);
        v.x += x.x; v.y += x.y; v.z += x.z; v.w += x.w;
      }
      const int n = n0 + rr;
      if (n < N && j0 + 4 * q < d.Pp) *reinterpret_cast<float4 *>(p.b.U + ((size_t)t * N + n) * d.Pp + j0 + 4 * q) = v;
    }
  }
  cl.sync();
}

// ---------------------------------------------------------------------------------------------
// stage 2:  grid (nCT + 1, nRT2, Tl)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(OP_THREADS, 2) k_stage2(KParams p) {
  extern __shared__ __align__(16) unsigned char dsm2[];
  Smem2 &sm = *reinterpret_cast<Smem2 *>(dsm2);
  const Dims &d = p.d;
  const int t = blockIdx.z, rt = blockIdx.y, ct = blockIdx.x, tid = threadIdx.x;
  const int N = d.N, D = d.D, P = d.P, C = d.C;
  const float *__restrict__ phi = p.phi + (size_t)t * d.phi_task_stride;
  const int d0 = rt * BR;
  const int nk = (N + BK - 1) / BK;
  const double beta = p.beta;

  // A tile: Φ[k0 + kk][d0 + 4q .. +3] → A[kk][4q..]  (2 × cp.async per thread)
  auto loadA = [&](int buf, int k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * OP_THREADS, kk = idx >> 5, q = idx & 31;
      const int n = k0 + kk, dd = d0 + 4 * q;
      const bool ok = n < N && dd < D;
      cp_async16(&sm.A[buf][kk][4 * q], ok ? phi + (size_t)n * D + dd : phi, ok);
    }
  };

  if (ct == d.nCT) {
    // ---------------- fp64 mean-column tile ---------------------------------------------------
    int any = 0;
    for (int c = 0; c < C; ++c) any |= (p.b.flagm[t * C + c] == 1);
    if (!any) return;
    const int r = tid & (BR - 1), h = tid >> 7;
    double acc[MAXC / 2];
#pragma unroll
    for (int i = 0; i < MAXC / 2; ++i) acc[i] = 0.0;
    auto loadB = [&](int buf, int k0) {
      if (tid < BK * C) {
        const int kk = tid / C, c = tid % C;
        sm.Bm[buf][kk][c] = (k0 + kk < N) ? p.b.Um[((size_t)t * N + k0 + kk) * C + c] : 0.0;
      }
    };
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
      if (s < nk) { loadA(s, s * BK); loadB(s, s * BK); }
      cp_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
      cp_wait<ST - 2>();
      __syncthreads();
      const int nx = kc + ST - 1;
      if (nx < nk) { loadA(nx % ST, nx * BK); loadB(nx % ST, nx * BK); }
      cp_commit();
      const int buf = kc % ST;
#pragma unroll 4
      for (int kk = 0; kk < BK; ++kk) {
        const double a = (double)sm.A[buf][kk][r];
#pragma unroll
        for (int i = 0; i < MAXC / 2; ++i)
          if (h + 2 * i < C) acc[i] = fma(a, sm.Bm[buf][kk][h + 2 * i], acc[i]);
      }
    }
    cp_wait<0>();
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
        const double wv = fma(beta, acc[i], p.b.alpha64[(size_t)c * D + dd] * dv);
        p.b.Wm[o] = wv;
        dot[i] = dv * wv;
      }
    }
    const int lane = tid & 31, wq = (tid >> 5) & 3;
#pragma unroll
    for (int i = 0; i < MAXC / 2; ++i) {
      double v = dot[i];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) sm.red[h][wq][i] = v;
    }
    __syncthreads();
    if (tid < MAXC) {
      const int hh = tid & 1, i = tid >> 1, c = hh + 2 * i;
      if (c < C) {
        double v = 0.0;
        for (int q = 0; q < 4; ++q) v += sm.red[hh][q][i];
        p.b.dAdm[((size_t)t * C + c) * d.nRT2 + rt] = v;
      }
    }
    if (tid == 0) atomicMax(p.b.ts + 4 * (*p.b.u) + 1, globaltimer());
    return;
  }

  // ---------------- fp32 probe tile -------------------------------------------------------
  const int m = p.b.m_act[t];
  const int j0 = ct * BC;
  if (j0 >= m) return;
  const int w = tid >> 5, l = tid & 31;
  const bool wact = j0 + w * WC < m;
  // B tile: U[t][k0 + kk][j0 + 4q .. +3] → B[kk][4q..]  (cp.async; 384 float4: kk = idx / 24, q = idx % 24)
  // columns ≥ m hold stale values: they only feed accumulators that are never stored
  auto loadB = [&](int buf, int k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * OP_THREADS, kk = idx / (BC / 4), q = idx % (BC / 4);
      if (idx < BK * BC / 4) {
        const int n = k0 + kk, j = j0 + 4 * q;
        const bool ok = n < N && j < d.Pp;
        cp_async16(&sm.B[buf][kk][4 * q], ok ? p.b.U + ((size_t)t * N + n) * d.Pp + j : p.b.U, ok);
      }
    }
  };
  float acc[4][WC];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < WC; ++c) acc[i][c] = 0.f;
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nk) { loadA(s, s * BK); loadB(s, s * BK); }
    cp_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_wait<ST - 2>();
    __syncthreads();
    const int nx = kc + ST - 1;
    if (nx < nk) { loadA(nx % ST, nx * BK); loadB(nx % ST, nx * BK); }
    cp_commit();
    const int buf = kc % ST;
    if (wact) {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        const float4 a = *reinterpret_cast<const float4 *>(&sm.A[buf][kk][4 * l]);
        const float *brow = &sm.B[buf][kk][w * WC];
        const float4 b0 = *reinterpret_cast<const float4 *>(brow);
        const float4 b1 = *reinterpret_cast<const float4 *>(brow + 4);
        const float4 b2 = *reinterpret_cast<const float4 *>(brow + 8);
        const float b[WC] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int c = 0; c < WC; ++c) acc[i][c] = fmaf(av[i], b[c], acc[i][c]);
      }
    }
  }
  cp_wait<0>();
  if (!wact) return;
  // epilogue: W = β acc + α_c ⊙ d for rows d0 + 4l .. +3, partial dᵀW (fp64) per column
  const float betaf = (float)beta;
  const int dd = d0 + 4 * l;
#pragma unroll
  for (int c = 0; c < WC; ++c) {
    const int j = j0 + w * WC + c;
    double dot = 0.0;
    int col = -1;
    if (j < m) {
      col = p.b.act[(size_t)t * P + j];
      if (dd < D) {
        const size_t base = ((size_t)t * P + col) * D;
        const float4 dv = ld4(p.b.Dv + base + dd);
        const float4 a4 = ld4(p.b.alpha32 + (size_t)(col / d.K) * D + dd);
        float4 wv;
        wv.x = fmaf(betaf, acc[0][c], a4.x * dv.x);
        wv.y = fmaf(betaf, acc[1][c], a4.y * dv.y);
        wv.z = fmaf(betaf, acc[2][c], a4.z * dv.z);
        wv.w = fmaf(betaf, acc[3][c], a4.w * dv.w);
        *reinterpret_cast<float4 *>(p.b.W + base + dd) = wv;
        dot = (double)dv.x * wv.x + (double)dv.y * wv.y + (double)dv.z * wv.z + (double)dv.w * wv.w;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (l == 0 && col >= 0) p.b.dAd[((size_t)t * P + col) * d.nRT2 + rt] = dot;
  }
  if (tid == 0) atomicMax(p.b.ts + 4 * (*p.b.u) + 1, globaltimer());  // warp 0 is always active here
}

}  // namespace

cudaError_t launch_stage1(const KParams &p, const double *mu_src, bool mu_only, cudaStream_t s) {
  const size_t smem = sizeof(Smem1) + sizeof(int) * (size_t)p.d.P;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(k_stage1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.d.nCT + 1, p.d.nRT1 * p.d.S1, p.d.Tl);
  cfg.blockDim = dim3(OP_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = p.d.S1;   // the split-K CTAs of one output tile form a cluster
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_stage1, p, mu_src ? mu_src : p.b.Dm, (int)(mu_only ? 1 : 0));
}

cudaError_t launch_stage2(const KParams &p, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_stage2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem2));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(p.d.nCT + 1, p.d.nRT2, p.d.Tl);
  k_stage2<<<grid, OP_THREADS, sizeof(Smem2), s>>>(p);
  return cudaGetLastError();
}

}  // namespace cmtcs
