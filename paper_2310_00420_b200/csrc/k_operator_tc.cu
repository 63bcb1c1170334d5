// K1 (probe columns) — the batched normal operator W = βΦ_tᵀ(Φ_t D) + α_{c(m)} ⊙ D on the 5th-gen
// tensor cores ("A := βΦᵀΦ + diag(α)", "solve all TC(K+1) systems
// simultaneously ... A never needs to be explicitly computed").  ΦᵀΦ is never formed.
//
//   stage 1  U[t][j][n] = Σ_d Φ_t[n][d] · D[t][act_j][d]        (M = 128 rows n, K = D, N = active cols)
//   stage 2  W[t][act_j][d] = β Σ_n Φ_t[n][d] · U[t][j][n] + α ⊙ D  (M = 128 rows d, K = N)
//            + fp64 partial dᵀ(Ad) per 128-row tile (Alg. 1 line 3)
//
// fp32-accurate products from TF32 tensor cores (3xTF32): every operand x is stored as an exact
// pair x = hi + lo with hi = tf32(x) and lo = x − hi, and each K = 8 step issues
//   acc_x += lo_A·hi_B + hi_A·lo_B ;  acc_m += hi_A·hi_B
// into separate TMEM accumulators (acc_x, acc_m), themselves split over K into `nacc` pairs and
// summed in fp32 in the epilogue — the tensor pipe's accumulation otherwise loses ~4 bits over
// long K (tools/tc_gemm_test.cu measures 3.2e-5 → 5e-6 relative at K = 4096; fp32 serial: 2e-6).
//
// One CTA = 128 threads computes a 128 × NT tile (NT ≤ 256 = column tile width; the MMA N is the
// tile's active column count rounded up to 16, so retired columns cost nothing).  Operands stream
// through an S-stage ring of 128-byte-swizzled K-major smem tiles: Φ and U tiles by TMA
// (cp.async.bulk.tensor), the gathered active direction columns of stage 1 by cp.async;
// thread 0 issues tcgen05.mma, tcgen05.commit frees a stage, tcgen05.ld drains TMEM.
// Stage 1 splits K over S1 CTAs for small T·N; the split CTAs form a thread-block cluster and
// reduce their partial tiles over DSMEM in fixed order (deterministic).
#include <cooperative_groups.h>

#include "cmtcs_internal.cuh"
#include "umma.cuh"

namespace cg = cooperative_groups;

namespace cmtcs {

using namespace umma;

namespace {

constexpr int TM = 128;                   // tile rows (MMA M)
constexpr int TK = 32;                    // K per pipeline stage (one 128-byte swizzled row)
constexpr uint32_t A_BYTES = TM * 128;    // 16 KB per hi / lo A tile
constexpr int MAXST = 4;

struct TcSmemTail {
  uint64_t full[MAXST], empty[MAXST];
  uint32_t tslot;
  int m;
  int act[256];        // the tile's active columns
  long long off[256];  // stage 2: element offset of column j's vectors, ((t·P + col)·D)
  int aoff[256];       // stage 2: offset of the column's α row, c·D
  double red[4][TC_NTMAX + MAXC];  // probe columns [0, NT), mean columns [TC_NTMAX, +C)
};

// Sums v[0..15] over the 32 lanes of a warp with 16 shuffles (butterfly transpose-reduce); the
// total of value index `idx` ends in the even lane with idx = bits 4..1 of the lane id.
__device__ __forceinline__ double warp_reduce16(double *v, int lane, int *idx) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool up = lane & 16;
    const double send = up ? v[i] : v[i + 8], keep = up ? v[i + 8] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool up = lane & 8;
    const double send = up ? v[i] : v[i + 4], keep = up ? v[i + 4] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool up = lane & 4;
    const double send = up ? v[i] : v[i + 2], keep = up ? v[i + 2] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  {
    const bool up = lane & 2;
    const double send = up ? v[0] : v[1], keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  *idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
  return v[0];
}

__device__ __forceinline__ unsigned char *stage_base(unsigned char *sm, int st, uint32_t stage_bytes) {
  return sm + (size_t)st * stage_bytes;
}

// TMEM accumulator column of pair q, term x (0 = main hi·hi, 1 = cross terms)
__device__ __forceinline__ uint32_t acc_col(int q, int x, int slot) { return (uint32_t)((2 * q + x) * slot); }

// issue the 3xTF32 MMAs of one K = 32 stage (thread 0 only)
__device__ __forceinline__ void mma_stage(uint32_t tmem, unsigned char *base, uint32_t b_bytes, uint32_t idesc,
                                          int q, int slot, bool first_of_acc) {
  const uint64_t ah = desc_sw128(smem_u32(base)), al = desc_sw128(smem_u32(base + A_BYTES));
  const uint64_t bh = desc_sw128(smem_u32(base + 2 * A_BYTES));
  const uint64_t bl = desc_sw128(smem_u32(base + 2 * A_BYTES + b_bytes));
  const uint32_t tm_m = tmem + acc_col(q, 0, slot), tm_x = tmem + acc_col(q, 1, slot);
#pragma unroll
  for (int k8 = 0; k8 < TK / 8; ++k8) {
    const uint64_t o = (uint64_t)(k8 * 32) >> 4;  // +32 bytes per K = 8 step inside the swizzled row
    const uint32_t acc = (first_of_acc && k8 == 0) ? 0u : 1u;
    mma_tf32(tm_x, al + o, bh + o, idesc, acc);
    mma_tf32(tm_x, ah + o, bl + o, idesc, 1u);
    mma_tf32(tm_m, ah + o, bh + o, idesc, acc);
  }
}

// 16 accumulator columns [c0, c0+16) of this thread's row, summed over the K-split pairs
__device__ __forceinline__ void acc_load16(uint32_t tmem, int warp, int c0, int nacc, int slot, float *tot) {
#pragma unroll
  for (int i = 0; i < 16; ++i) tot[i] = 0.f;
  for (int x = 1; x >= 0; --x)        // cross terms first, then the main products
    for (int q = 0; q < nacc; ++q) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + acc_col(q, x, slot) + c0, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) tot[i] += v[i];
    }
}

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

// fp64 mean-column work on the A tile already in smem (CUDA cores, while the tensor core runs):
// acc[c] += Σ_{k in stage} Φ[r][k] · B[c][k] for this thread's row r, Φ = hi + lo (exact in fp32).
// Stage 1 reads B as [c][k] (k contiguous), stage 2 as [k][c].
template <bool B_CK>
__device__ __forceinline__ void mean_stage(const unsigned char *base, const double *mb, int r, int C, double *acc) {
#pragma unroll
  for (int cc = 0; cc < TK / 4; ++cc) {
    const float4 h = *reinterpret_cast<const float4 *>(base + sw128_offset(r, cc));
    const float4 l = *reinterpret_cast<const float4 *>(base + A_BYTES + sw128_offset(r, cc));
    const double a[4] = {(double)(h.x + l.x), (double)(h.y + l.y), (double)(h.z + l.z), (double)(h.w + l.w)};
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      if (c < C) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double bv = B_CK ? mb[c * TK + 4 * cc + i] : mb[(4 * cc + i) * C + c];
          acc[c] = fma(a[i], bv, acc[c]);
        }
      }
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t *mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}

// ---------------------------------------------------------------------------------------------
// stage 1:  grid (nCT, nRT1 * S1, Tl), cluster (1, S1, 1), 128 threads
//   probe columns: U = Φ·D on the tensor core (3xTF32);  column tile 0 also computes the fp64
//   mean columns Um = Φ·Dm on the CUDA cores from the same smem Φ tiles.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_stage1_tc(KParams p, const __grid_constant__ CUtensorMap tPhiH, const __grid_constant__ CUtensorMap tPhiL) {
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~(uintptr_t)1023);
  const Dims &d = p.d;
  const TcCfg &tc = p.tc;
  TcSmemTail &tl = *reinterpret_cast<TcSmemTail *>(sm + (size_t)tc.stages * tc.stage_bytes);
  int *s_all = reinterpret_cast<int *>(&tl + 1);  // full act list of the task (P entries)
  const int t = blockIdx.z, ct = blockIdx.x, tid = threadIdx.x, warp = tid >> 5;
  const int rt = blockIdx.y / d.S1, sp = blockIdx.y % d.S1;
  const int N = d.N, D = d.D, P = d.P, C = d.C;
  const int u = *p.b.u;
  if (u >= d.cap) return;                     // past the end of an unrolled graph body
  if (tid == 0) atomicMax(p.b.ts + 4 * u, ~globaltimer());  // ~t: max ⇔ min
  const int m = build_act(p.b.flag + (size_t)t * P, P, s_all, &tl.m);
  int mc = 0;
  for (int c = 0; c < C; ++c) mc += (p.b.flagm[t * C + c] == 1);
  if (ct == 0 && blockIdx.y == 0 && tid == 0) {
    // task bookkeeping for this CG step: publish the act list and the step histograms
    p.b.m_act[t] = m;
    if (m) atomicAdd(p.b.hist + u, m);
    if (mc) atomicAdd(p.b.histm + u, mc);
    if (m + mc) atomicAdd(p.b.histt + u, 1);
  }
  if (ct == 0 && blockIdx.y == 0)
    for (int j = tid; j < m; j += TC_THREADS) p.b.act[(size_t)t * P + j] = s_all[j];
  const int j0 = ct * tc.NT;
  const bool run_probe = j0 < m, run_mean = ct == 0 && mc > 0;
  if (!run_probe && !run_mean) return;        // cluster-uniform (same t, ct)
  const int ncol = run_probe ? min(tc.NT, m - j0) : 0;
  const int nmma = (ncol + 15) & ~15;
  const int n0 = rt * TM;
  const int kb = sp * d.K1, ke = min(D, kb + d.K1);
  const int nk = (ke - kb + TK - 1) / TK;
  const int arow = (d.shared_phi ? 0 : t * N) + n0;
  const uint32_t b_bytes = (uint32_t)tc.NT * 128;
  const uint32_t mu_off = 2 * A_BYTES + 2 * b_bytes;   // fp64 mean-column chunk [C][32]
  const int slot = tc.slot, nacc = min(tc.nacc, nk), S = tc.stages;  // every pair gets ≥ 1 chunk
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&tl.full[s], 1); mbar_init(&tl.empty[s], 1); }
    fence_mbar_init();
    prefetch_tmap(&tPhiH);
    prefetch_tmap(&tPhiL);
  }
  if (warp == 0 && nmma) tmem_alloc<512>(&tl.tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tl.tslot;
  const uint32_t idesc = idesc_tf32(TM, nmma > 0 ? nmma : 16);
  const float *Dh = p.b.Dh + (size_t)t * P * D, *Dl = p.b.Dl + (size_t)t * P * D;
  const double *Dm = p.b.Dm + (size_t)t * C * D;

  auto issue = [&](int st, int kc) {
    unsigned char *base = stage_base(sm, st, tc.stage_bytes);
    const int k0 = kb + kc * TK;
    if (tid == 0) {
      mbar_arrive_expect_tx(&tl.full[st], 2 * A_BYTES);
      tma_load_2d(base, &tPhiH, k0, arow, &tl.full[st]);
      tma_load_2d(base + A_BYTES, &tPhiL, k0, arow, &tl.full[st]);
    }
    // gather the active direction columns (hi, lo): nmma rows x 8 chunks of 16 bytes
    const uint32_t sb = smem_u32(base + 2 * A_BYTES);
    for (int e = tid; e < nmma * 8; e += TC_THREADS) {
      const int j = e >> 3, c = e & 7;
      const int k = k0 + 4 * c;
      const bool ok = j < ncol && k < ke;
      const size_t off = ok ? (size_t)s_all[j0 + j] * D + k : 0;
      cp_async16(sb + sw128_offset(j, c), Dh + off, ok);
      cp_async16(sb + b_bytes + sw128_offset(j, c), Dl + off, ok);
    }
    if (run_mean)                             // Dm[c][k0 .. k0+31] → [c][k], 2 doubles per copy
      for (int e = tid; e < C * (TK / 2); e += TC_THREADS) {
        const int c = e / (TK / 2), k2 = e % (TK / 2);
        const int k = k0 + 2 * k2;
        const bool ok = k < ke;
        cp_async16(smem_u32(base + mu_off) + (uint32_t)(c * TK + 2 * k2) * 8, ok ? Dm + (size_t)c * D + k : Dm, ok);
      }
  };
  double macc[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) macc[c] = 0.0;
  const int r = warp * 32 + (tid & 31);       // tile row = TMEM lane
  for (int s = 0; s < S - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    const int st = kc % S;
    mbar_wait(&tl.full[st], (kc / S) & 1);
    cp_wait_dyn(S - 2);
    fence_proxy_async();
    __syncthreads();
    unsigned char *base = stage_base(sm, st, tc.stage_bytes);
    if (tid == 0) {
      if (nmma) {
        fence_after_sync();
        const int q = (kc * nacc) / nk;
        const int qfirst = (q * nk + nacc - 1) / nacc;
        mma_stage(tmem, base, b_bytes, idesc, q, slot, kc == qfirst);
        mma_commit(&tl.empty[st]);
      } else {
        mbar_arrive(&tl.empty[st]);
      }
    }
    if (run_mean) mean_stage<true>(base, reinterpret_cast<const double *>(base + mu_off), r, C, macc);
    const int nx = kc + S - 1;
    if (nx < nk) {
      const int ns = nx % S;
      if (nx >= S) mbar_wait(&tl.empty[ns], ((nx - S) / S) & 1);
      __syncthreads();                        // every thread is done reading stage ns (mean part)
      issue(ns, nx);
    }
    cp_commit();
  }
  mbar_wait(&tl.empty[(nk - 1) % S], ((nk - 1) / S) & 1);
  fence_after_sync();

  const int n = n0 + r;
  float *Uh = p.b.Uh + (size_t)t * d.Pp * N, *Ul = p.b.Ul + (size_t)t * d.Pp * N;
  if (d.S1 == 1) {
    for (int c0 = 0; c0 < nmma; c0 += 16) {
      float tot[16];
      acc_load16(tmem, warp, c0, nacc, slot, tot);
      if (n < N) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = j0 + c0 + i;
          if (c0 + i < ncol) {
            const float h = tf32_hi(tot[i]);
            Uh[(size_t)j * N + n] = h;
            Ul[(size_t)j * N + n] = tot[i] - h;
          }
        }
      }
    }
    if (run_mean && n < N) {
#pragma unroll
      for (int c = 0; c < MAXC; ++c)
        if (c < C) p.b.Um[((size_t)t * N + n) * C + c] = macc[c];
    }
  } else {
    // split-K: partial tiles in smem (aliases the drained ring), cluster DSMEM reduction
    __syncthreads();
    float *part = reinterpret_cast<float *>(sm);                         // [NT][128] fp32
    double *partm = reinterpret_cast<double *>(sm + (size_t)tc.NT * TM * 4);  // [128][MAXC] fp64
    for (int c0 = 0; c0 < nmma; c0 += 16) {
      float tot[16];
      acc_load16(tmem, warp, c0, nacc, slot, tot);
#pragma unroll
      for (int i = 0; i < 16; ++i) part[(c0 + i) * TM + r] = tot[i];
    }
    if (run_mean) {
#pragma unroll
      for (int c = 0; c < MAXC; ++c)
        if (c < C) partm[r * MAXC + c] = macc[c];
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int rows = TM / d.S1, rb = sp * rows;
    for (int e = tid; e < rows * ncol; e += TC_THREADS) {
      const int c = e / rows, rr = rb + e % rows;
      float v = 0.f;
      for (int src = 0; src < d.S1; ++src) v += cl.map_shared_rank(part, src)[c * TM + rr];  // fixed order
      const int nn = n0 + rr;
      if (nn < N) {
        const float h = tf32_hi(v);
        Uh[(size_t)(j0 + c) * N + nn] = h;
        Ul[(size_t)(j0 + c) * N + nn] = v - h;
      }
    }
    if (run_mean)
      for (int e = tid; e < rows * C; e += TC_THREADS) {
        const int rr = rb + e / C, c = e % C;
        double v = 0.0;
        for (int src = 0; src < d.S1; ++src) v += cl.map_shared_rank(partm, src)[rr * MAXC + c];
        if (n0 + rr < N) p.b.Um[((size_t)t * N + n0 + rr) * C + c] = v;
      }
    cl.sync();
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0 && nmma) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------------------------
// stage 2:  grid (nCT, nRT2, Tl), 128 threads
//   probe columns: W = βΦᵀU + α⊙D (tensor core) and fp64 partial dᵀW;  column tile 0 also the fp64
//   mean columns Wm = βΦᵀUm + α⊙Dm and dᵀW partials on the CUDA cores from the same Φᵀ tiles.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_stage2_tc(KParams p, const __grid_constant__ CUtensorMap tPtH, const __grid_constant__ CUtensorMap tPtL,
                const __grid_constant__ CUtensorMap tUH, const __grid_constant__ CUtensorMap tUL) {
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~(uintptr_t)1023);
  const Dims &d = p.d;
  const TcCfg &tc = p.tc;
  TcSmemTail &tl = *reinterpret_cast<TcSmemTail *>(sm + (size_t)tc.stages * tc.stage_bytes);
  const int t = blockIdx.z, ct = blockIdx.x, rt = blockIdx.y, tid = threadIdx.x, warp = tid >> 5;
  const int N = d.N, D = d.D, P = d.P, C = d.C;
  if (*p.b.u >= d.cap) return;
  const int m = p.b.m_act[t];
  int mc = 0;
  for (int c = 0; c < C; ++c) mc += (p.b.flagm[t * C + c] == 1);
  const int j0 = ct * tc.NT;
  const bool run_probe = j0 < m, run_mean = ct == 0 && mc > 0;
  if (!run_probe && !run_mean) return;
  const int ncol = run_probe ? min(tc.NT, m - j0) : 0;
  const int nmma = (ncol + 15) & ~15;
  const int d0 = rt * TM;
  const int nk = (N + TK - 1) / TK;
  const int arow = (d.shared_phi ? 0 : t * D) + d0;
  const int brow = t * d.Pp + j0;
  const uint32_t b_bytes = (uint32_t)tc.NT * 128;
  const uint32_t mu_off = 2 * A_BYTES + 2 * b_bytes;   // fp64 mean-column chunk [32][C]
  const int slot = tc.slot, nacc = min(tc.nacc, nk), S = tc.stages;  // every pair gets ≥ 1 chunk
  for (int j = tid; j < ncol; j += TC_THREADS) {
    const int col = p.b.act[(size_t)t * P + j0 + j];
    tl.act[j] = col;
    tl.off[j] = ((long long)t * P + col) * D;
    tl.aoff[j] = (col / d.K) * D;
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&tl.full[s], 1); mbar_init(&tl.empty[s], 1); }
    fence_mbar_init();
    prefetch_tmap(&tPtH);
    prefetch_tmap(&tPtL);
    prefetch_tmap(&tUH);
    prefetch_tmap(&tUL);
  }
  if (warp == 0 && nmma) tmem_alloc<512>(&tl.tslot);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tl.tslot;
  const uint32_t idesc = idesc_tf32(TM, nmma > 0 ? nmma : 16);
  const double *Um = p.b.Um + (size_t)t * N * C;

  auto issue = [&](int st, int kc) {
    unsigned char *base = stage_base(sm, st, tc.stage_bytes);
    const int k0 = kc * TK;
    if (tid == 0) {
      mbar_arrive_expect_tx(&tl.full[st], 2 * A_BYTES + (nmma ? 2 * b_bytes : 0));
      tma_load_2d(base, &tPtH, k0, arow, &tl.full[st]);
      tma_load_2d(base + A_BYTES, &tPtL, k0, arow, &tl.full[st]);
      if (nmma) {
        tma_load_2d(base + 2 * A_BYTES, &tUH, k0, brow, &tl.full[st]);
        tma_load_2d(base + 2 * A_BYTES + b_bytes, &tUL, k0, brow, &tl.full[st]);
      }
    }
    if (run_mean) {                            // Um[k0 .. k0+31][0..C) is contiguous: 32·C 8-byte copies
      for (int e = tid; e < C * TK; e += TC_THREADS) {
        const bool ok = k0 + e / C < N;
        cp_async8(smem_u32(base + mu_off) + (uint32_t)e * 8, ok ? Um + (size_t)k0 * C + e : Um, ok);
      }
    }
  };
  double macc[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) macc[c] = 0.0;
  const int r = warp * 32 + (tid & 31);
  for (int s = 0; s < S - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    const int st = kc % S;
    mbar_wait(&tl.full[st], (kc / S) & 1);
    cp_wait_dyn(S - 2);
    fence_proxy_async();
    __syncthreads();
    unsigned char *base = stage_base(sm, st, tc.stage_bytes);
    if (tid == 0) {
      if (nmma) {
        fence_after_sync();
        const int q = (kc * nacc) / nk;
        const int qfirst = (q * nk + nacc - 1) / nacc;
        mma_stage(tmem, base, b_bytes, idesc, q, slot, kc == qfirst);
        mma_commit(&tl.empty[st]);
      } else {
        mbar_arrive(&tl.empty[st]);
      }
    }
    if (run_mean) mean_stage<false>(base, reinterpret_cast<const double *>(base + mu_off), r, C, macc);
    const int nx = kc + S - 1;
    if (nx < nk) {
      const int ns = nx % S;
      if (nx >= S) mbar_wait(&tl.empty[ns], ((nx - S) / S) & 1);
      __syncthreads();                        // every thread is done reading stage ns (mean part)
      issue(ns, nx);
    }
    cp_commit();
  }
  mbar_wait(&tl.empty[(nk - 1) % S], ((nk - 1) / S) & 1);
  fence_after_sync();

  // epilogue: W = β acc + α_c ⊙ d for row dd, fp64 partial dᵀW per column (this 128-row tile).
  // Per group of 16 columns all global loads are issued first, then the math, then a butterfly
  // reduction of the 16 dot partials over the warp.
  const int dd = d0 + r;
  const bool rv = dd < D;
  const float betaf = (float)p.beta;
  const int lane = tid & 31;
  for (int c0 = 0; c0 < nmma; c0 += 16) {
    float tot[16], dh[16], dl[16], al[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const bool ok = c0 + i < ncol && rv;
      const long long o = ok ? tl.off[c0 + i] + dd : 0;
      dh[i] = ok ? p.b.Dh[o] : 0.f;
      dl[i] = ok ? p.b.Dl[o] : 0.f;
      al[i] = ok ? p.b.alpha32[tl.aoff[c0 + i] + dd] : 0.f;
    }
    acc_load16(tmem, warp, c0, nacc, slot, tot);
    double dot[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float dv = dh[i] + dl[i];
      const float w = fmaf(betaf, tot[i], al[i] * dv);
      if (c0 + i < ncol && rv) p.b.W[tl.off[c0 + i] + dd] = w;
      dot[i] = (double)dv * (double)w;
    }
    int idx;
    const double sum = warp_reduce16(dot, lane, &idx);
    if ((lane & 1) == 0) tl.red[warp][c0 + idx] = sum;
  }
  if (run_mean) {
    // mean columns (fp64): Wm = β·acc + α ⊙ dm, partial dᵀWm over this row tile
    double dot[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      dot[c] = 0.0;
      if (c < C && rv) {
        const size_t o = ((size_t)t * C + c) * D + dd;
        const double dmv = p.b.Dm[o];
        const double wv = fma(p.beta, macc[c], p.b.alpha64[(size_t)c * D + dd] * dmv);
        p.b.Wm[o] = wv;
        dot[c] = dmv * wv;
      }
    }
    int idx;
    const double sum = warp_reduce16(dot, lane, &idx);
    if ((lane & 1) == 0 && idx < C) tl.red[warp][TC_NTMAX + idx] = sum;
  }
  fence_before_sync();
  __syncthreads();
  for (int jj = tid; jj < ncol; jj += TC_THREADS)
    p.b.dAd[((size_t)t * P + tl.act[jj]) * d.nRT2 + rt] = tl.red[0][jj] + tl.red[1][jj] + tl.red[2][jj] + tl.red[3][jj];
  if (run_mean && tid < C) {
    const int jj = TC_NTMAX + tid;
    p.b.dAdm[((size_t)t * C + tid) * d.nRT2 + rt] = tl.red[0][jj] + tl.red[1][jj] + tl.red[2][jj] + tl.red[3][jj];
  }
  if (tid == 0) atomicMax(p.b.ts + 4 * (*p.b.u) + 1, globaltimer());
  if (warp == 0 && nmma) tmem_dealloc<512>(tmem);
}

// Φ → (Φhi, Φlo) and the transposed pair (Φᵀhi, Φᵀlo), once at init.  32×32 smem-tiled transpose.
__global__ void k_split_phi(const float *__restrict__ phi, int rows, int cols, int mats, float *hi, float *lo,
                            float *thi, float *tlo) {
  __shared__ float tile[32][33];
  const int mat = blockIdx.z;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const float *src = phi + (size_t)mat * rows * cols;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    float v = 0.f;
    if (r < rows && c < cols) {
      v = src[(size_t)r * cols + c];
      const float h = tf32_hi(v);
      hi[(size_t)mat * rows * cols + (size_t)r * cols + c] = h;
      lo[(size_t)mat * rows * cols + (size_t)r * cols + c] = v - h;
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;   // transposed: row c, column r
    if (c < cols && r < rows) {
      const float v = tile[threadIdx.x][i];
      const float h = tf32_hi(v);
      thi[(size_t)mat * rows * cols + (size_t)c * rows + r] = h;
      tlo[(size_t)mat * rows * cols + (size_t)c * rows + r] = v - h;
    }
  }
}

}  // namespace

size_t tc_smem_bytes(const TcCfg &tc, int P) {
  return 1024 + (size_t)tc.stages * tc.stage_bytes + sizeof(TcSmemTail) + sizeof(int) * (size_t)P;
}

cudaError_t launch_split_phi(const KParams &p, cudaStream_t s) {
  const int mats = p.d.shared_phi ? 1 : p.d.Tl;
  dim3 grid((p.d.D + 31) / 32, (p.d.N + 31) / 32, mats);
  k_split_phi<<<grid, dim3(32, 8), 0, s>>>(p.phi, p.d.N, p.d.D, mats, p.b.Phh, p.b.Phl, p.b.PTh, p.b.PTl);
  return cudaGetLastError();
}

cudaError_t launch_stage1_tc(const KParams &p, const TcMaps &maps, cudaStream_t s) {
  const size_t smem = tc_smem_bytes(p.tc, p.d.P);
  cudaError_t e = cudaFuncSetAttribute(k_stage1_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.d.nCT, p.d.nRT1 * p.d.S1, p.d.Tl);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = p.d.S1;   // the split-K CTAs of one output tile form a cluster
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_stage1_tc, p, maps.phi_h, maps.phi_l);
}

cudaError_t launch_stage2_tc(const KParams &p, const TcMaps &maps, cudaStream_t s) {
  const size_t smem = tc_smem_bytes(p.tc, p.d.P);
  cudaError_t e = cudaFuncSetAttribute(k_stage2_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_stage2_tc<<<dim3(p.d.nCT, p.d.nRT2, p.d.Tl), TC_THREADS, smem, s>>>(p, maps.phit_h, maps.phit_l, maps.u_h,
                                                                        maps.u_l);
  return cudaGetLastError();
}

}  // namespace cmtcs
