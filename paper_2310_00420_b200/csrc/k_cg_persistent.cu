// The batched conjugate-gradient loop of one E-step (Alg. 1, run for every task t,
// cluster c and right-hand side of Alg. 2 lines 5-6) as ONE persistent kernel:
// one CTA per SM, all CG steps of the EM iteration inside, three grid-wide phases per step.
//
//   phase 1 (K1, stage 1)  U[t][j][n] = Σ_d Φ_t[n][d] · D[t][j][d]                tensor cores (3xTF32)
//   phase 2 (K1, stage 2)  W[t][j][d] = β Σ_n Φ_t[n][d] · U[t][j][n] + α_c ⊙ D   (PAPER.md:80, 157:
//                          "A := βΦᵀΦ + diag(α)", ΦᵀΦ never formed) + fp64 partials of dᵀW
//                          (dᵀAd is formed from the same W the residual update subtracts: computing it
//                          as β‖Φd‖² + dᵀdiag(α)d instead is algebraically equal but inconsistent with
//                          the rounded W, and measured 20x worse log-likelihood parity at C2)
//   phase 3 (K4, update)   γ_u = rᵀr / dᵀAd; x += γd; r −= γAd; ξ_u = r'ᵀr'/rᵀr; d = r' + ξd;
//                          convergence ‖r'‖ ≤ tol·‖b‖ (reading A5); transcript (γ_u, ξ_u)
//
// Phases are separated by a grid barrier (all CTAs co-resident: cooperative launch, one CTA per
// SM); the work units of a phase (output tiles, columns) are dealt round-robin to the CTAs.  The
// C fp64 mean columns of a task ride along with the task's column-tile-0 units: fp64 DFMA on the
// CUDA cores, reading the same smem Φ tiles the tensor core reads.
//
// Warp roles in phases 1-2 (320 threads):
//   warp 0     TMA producer: fp32 Φ/Φᵀ tiles (A), direction / U tiles (B), fp64 mean-column chunk
//   warp 1     MMA issuer: tcgen05.mma kind::tf32 with A in TMEM, tcgen05.commit frees stages / tiles
//   warps 2-5  the A warps (one per TMEM lane quarter; warp 2 also owns TMEM): split every staged
//              fp32 A tile into the exact tf32 pair hi + lo and write it to a TMEM A stage
//              (tcgen05.st)
//   warps 6-9  the epilogue: the fp64 mean columns' DMMA on the staged fp32 tiles during a unit's
//              K loop (the FP64 pipe of each SM sub-partition, beside the A warps' split), then the
//              unit's outputs (TMEM → registers → U / W, dᵀAd partials); with double-buffered TMEM
//              accumulators the MMAs of the next unit run while the epilogue drains
// All operands arrive by TMA into an S-stage ring of 128-byte-swizzled K-major smem tiles, so no
// CTA-wide barrier runs inside a K loop; the producer runs ahead into the next unit while the
// epilogue of the previous one drains.  mbarriers: full[s] (TMA bytes), empty[s] (MMA done and the
// four A warps done with the stage), mdone[s] (the epilogue warps' fp64 work on a mean chunk done),
// afull[a] / aempty[a] (TMEM A stage written / consumed by the MMAs), tfull / tempty (accumulator
// handshake).
//
// The A operands (Φ itself and its transpose) live in HBM as plain fp32 and arrive by TMA; the A
// warps split each staged tile into hi = tf32(x), lo = x − hi straight into tensor memory, so the
// shared-memory port carries each A byte once (TMA write, one read) and the MMAs read only B from
// shared memory.  The B operands (directions, U — small next to Φ and re-read by every row tile)
// are written by their producers as tf32 pairs and staged as such.
//
// 3xTF32: every operand x is the exact pair x = hi + lo with hi = tf32(x), and each K = 8 step issues
//   acc_x += lo_A·hi_B + hi_A·lo_B ;  acc_m += hi_A·hi_B
// into separate TMEM accumulators, the main one split over K into up to 4 and summed in fp32 in
// the epilogue (the tensor pipe's accumulation otherwise loses ~4 bits over long K;
// tools/tc_gemm_test.cu measures 3.2e-5 → 5e-6 relative at K = 4096; fp32 serial FFMA: 2e-6).
//
// Columns are not compacted: a unit multiplies its whole column tile (retired columns included,
// their results are ignored) and is skipped when none of its columns is active.  Stage 1 may split
// the contraction over D (S1 > 1) to balance the grid; the S1 partial tiles are reduced through
// global memory by the last-arriving CTA of the tile, in fixed order (deterministic).
//
// Memory ordering: every phase boundary is a grid barrier whose acquire fence (fence.acq_rel.gpu,
// CCTL.IVALL in SASS) invalidates the SM's L1, so data written by other CTAs in earlier phases is
// read with ordinary loads; TMA reads of such data follow fence.proxy.async.  Split-K partials,
// exchanged within a phase, are read with ld.global.cg after the tile counter's acquire.
#include <stdio.h>

#include <algorithm>

#include "cmtcs_internal.cuh"
#include "umma.cuh"

namespace cmtcs {

using namespace umma;

namespace {

constexpr int TM = 128;                   // tile rows (MMA M)
constexpr int TK = 32;                    // K per pipeline stage (one 128-byte swizzled row)
constexpr uint32_t A_BYTES = TM * 128;    // 16 KB fp32 A tile per ring stage
constexpr int MAXST = 6;
constexpr int MAXSA = 4;                  // TMEM A stages
constexpr int NTHREADS = 320;
constexpr int AW0 = 64;                   // first thread of the A (split) warps 2-5
constexpr int EPI0 = 192;                 // first thread of the epilogue warps 6-9

struct PSmemTail {
  uint64_t full[MAXST], empty[MAXST], mdone[MAXST];
  uint64_t bfull[MAXST];                  // CTA pairs: both CTAs' B halves landed (the leader's copy is used)
  uint64_t afull[MAXSA], aempty[MAXSA];   // TMEM A stages: written by the A warps / read by the MMAs
  uint64_t tfull[2], tempty[2];      // TMEM accumulator buffers: MMA done / epilogue drained
  uint64_t dfull, dempty;             // the stage-2 epilogue's d tile (TMA bytes / epilogue done)
  uint32_t tslot;
  uint32_t help_tacc;                 // the accumulator buffer of a tile drained by A + epilogue warps
  int last;                           // split-K: this CTA reduces the tile (last-arriver mode)
  uint32_t emask[4][TC_NTMAX / 32];   // per epilogue warp: active-column mask of its current tile
  double red[4][TC_NTMAX];            // per epilogue warp: dᵀAd partials of the probe columns
  double redm[4][MAXC];               // per mean warp: dᵀAd partials of the mean columns
};

template <class T>
__device__ __forceinline__ T ldv(const T *p) { return *p; }
template <class T>
__device__ __forceinline__ void stv(T *p, T v) { *p = v; }

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// TMA prefetch of an A tile into L2 (no shared memory, no completion tracking): the A operand (Φ /
// Φᵀ) streams from HBM once per step, and a ring of S stages holds too few bytes to cover that
// latency at the MMA rate (Little's law: ~200 KB in flight against ~2.4k clk from issue to landing)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}
// named barrier among the 4 epilogue warps
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 2, 128;\n" ::: "memory"); }
// named barrier among the A warps and the epilogue warps (a CTA's last stage-2 tile, drained by both)
__device__ __forceinline__ void pair_sync() { asm volatile("bar.sync 3, 256;\n" ::: "memory"); }

// grid-wide barrier over the co-resident CTAs: a monotonically increasing arrival counter
// (reset to 0 before every launch); epoch e completes when the counter reaches e·gridDim.x
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned &epoch) {
  // this thread's generic writes → later async-proxy accesses: global (TMA reads of d, U) and
  // shared (the update phase parks d / r in the idle ring, which the next step's TMA overwrites)
  asm volatile("fence.proxy.async;\n" ::: "memory");
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) {
    const unsigned target = epoch * gridDim.x;
    // the release is cumulative over the CTA's writes ordered before it by the barrier above
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    unsigned v;
    do {   // relaxed polling (no L1 invalidation per poll), one acquire fence once released
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  }
  __syncthreads();
}

// Per-task dataflow between the phases (instead of grid barriers): a unit's completion is released
// on its task's counter (the unit's stores fenced first), and a consumer acquires the counter until
// it reaches the step's target (units per task × (step + 1); skipped units count too).
__device__ __forceinline__ void dep_signal(int *cnt) {
  asm volatile("red.release.gpu.global.add.s32 [%0], 1;\n" ::"l"(cnt) : "memory");
}
__device__ __forceinline__ void dep_wait(const int *cnt, int target) {
  int v;
  do {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(cnt) : "memory");
  } while (v < target);
}

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

// The same in fp32 with an error-free product split: v = p + e exactly per element (p = d·w rounded,
// e = fma(d, w, −p)), the p's and e's butterflied separately (fp32 shuffles are one SHFL, fp64
// two, and the fp64 conversions cost as much as the MMAs: tools/dmma_test.cu); the total is
// returned in fp64 as p_sum + e_sum.
__device__ __forceinline__ double warp_reduce16_f(float *p, float *e, int lane, int *idx) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool up = lane & 16;
    const float sp = up ? p[i] : p[i + 8], kp = up ? p[i + 8] : p[i];
    const float se = up ? e[i] : e[i + 8], ke = up ? e[i + 8] : e[i];
    p[i] = kp + __shfl_xor_sync(0xffffffffu, sp, 16);
    e[i] = ke + __shfl_xor_sync(0xffffffffu, se, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool up = lane & 8;
    const float sp = up ? p[i] : p[i + 4], kp = up ? p[i + 4] : p[i];
    const float se = up ? e[i] : e[i + 4], ke = up ? e[i + 4] : e[i];
    p[i] = kp + __shfl_xor_sync(0xffffffffu, sp, 8);
    e[i] = ke + __shfl_xor_sync(0xffffffffu, se, 8);
  }
  // from here fp64: 4 → 1 values per lane pair, few conversions
  double pd[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) pd[i] = (double)p[i] + (double)e[i];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool up = lane & 4;
    const double send = up ? pd[i] : pd[i + 2], keep = up ? pd[i + 2] : pd[i];
    pd[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  {
    const bool up = lane & 2;
    const double send = up ? pd[0] : pd[1], keep = up ? pd[1] : pd[0];
    pd[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  pd[0] += __shfl_xor_sync(0xffffffffu, pd[0], 1);
  *idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
  return pd[0];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// TMEM accumulators of a tile: the cross terms (lo·hi + hi·lo, ~2^-11 of the product) in one
// accumulator at column 0, the main terms (hi·hi) split over K into `nacc` accumulators at columns
// (1 + q)·slot, summed in fp32 in the epilogue (the tensor pipe's fp32 accumulation loses bits over
// long K).  Short contractions (≤ 32 chunks, K ≤ 1024) use one main accumulator and two buffers
// of 2·slot columns (double buffering: the MMA warp starts the next tile while the epilogue drains
// this one) when they fit below the A stages; longer ones up to tc.nacc main accumulators.
// Double buffering only for short contractions (≤ 16 chunks, K ≤ 512): a longer K goes to K-split
// main accumulators instead — the tensor pipe's fp32 accumulation truncates, and the bias it leaves
// in Ad shifts the Lanczos log-det (ν̄, hence L) systematically: at C3 (stage 2, K = 1024) one
// accumulator measured |ΔL| = 1.06e-3 against the oracle, three 4.0e-4, for 2.5 % of the step
//
__device__ __forceinline__ bool unit_dbl(const TcCfg &tc, int nk, int dbg) {
  return tc.dbl && nk <= (dbg & 32 ? 64 : 16) && !(dbg & 16);
}
__device__ __forceinline__ int unit_nacc(const TcCfg &tc, int nk, int dbg) {
  if (unit_dbl(tc, nk, dbg)) return 1;
  return (nk <= 16 && !(dbg & 8)) ? 1 : min(tc.nacc, nk);
}

// issue the 3xTF32 MMAs of one K = 32 stage (the whole MMA warp, one elected lane issuing) into main
// accumulator q: A (hi | lo) from
// the TMEM A stage at column a_tm, B (hi, lo) from the shared-memory ring stage
// (CTA pairs: one cta_group::2 instruction covers both CTAs' 128 rows; each CTA's stage holds its
// half of the tile's columns, hi half then lo half, at the same offsets: lo_off = the hi half's bytes)
template <bool PR>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (PR) mma_tf32_ts_warp_pair(d, a, b, idesc, acc);
  else mma_tf32_ts_warp(d, a, b, idesc, acc);
}
template <bool PR>
__device__ __forceinline__ void mma_stage(uint32_t tmem, uint32_t a_tm, unsigned char *base, uint32_t lo_off,
                                          uint32_t idesc, int q, int slot, bool first_main, bool first_cross) {
  const uint64_t bh = desc_sw128(smem_u32(base + A_BYTES));
  const uint64_t bl = desc_sw128(smem_u32(base + A_BYTES + lo_off));
  const uint32_t tm_m = tmem + (uint32_t)((1 + q) * slot), tm_x = tmem;
#pragma unroll
  for (int k8 = 0; k8 < TK / 8; ++k8) {
    const uint64_t o = (uint64_t)(k8 * 32) >> 4;  // +32 bytes per K = 8 step inside the swizzled row
    const uint32_t ah = a_tm + 8 * k8, al = a_tm + 32 + 8 * k8;
    mma_ts<PR>(tm_x, al, bh + o, idesc, (first_cross && k8 == 0) ? 0u : 1u);
    mma_ts<PR>(tm_x, ah, bl + o, idesc, 1u);
    mma_ts<PR>(tm_m, ah, bh + o, idesc, (first_main && k8 == 0) ? 0u : 1u);
  }
}

// The same for a full double-buffered tile (N = NT, slot = NT, one main accumulator) in 2 MMAs per
// K = 8 step instead of 3: the B hi and lo tiles are adjacent in shared memory, so one N = 2·NT MMA
// computes hi_A·[hi_B | lo_B] into [main | cross] (columns [0, NT) and [NT, 2·NT) of the buffer, the
// same regions the 3-MMA form uses for cross and main — the epilogue sums both either way), and a
// second adds lo_A·hi_B to the cross region.  Fewer MMA instructions per chunk for the issuing warp.
__device__ __forceinline__ void mma_stage_cat(uint32_t tmem, uint32_t a_tm, unsigned char *base, uint32_t idesc2,
                                              uint32_t idesc, int nt, bool first) {
  const uint64_t bh = desc_sw128(smem_u32(base + A_BYTES));
#pragma unroll
  for (int k8 = 0; k8 < TK / 8; ++k8) {
    const uint64_t o = (uint64_t)(k8 * 32) >> 4;
    const uint32_t ah = a_tm + 8 * k8, al = a_tm + 32 + 8 * k8;
    mma_tf32_ts_warp(tmem, ah, bh + o, idesc2, (first && k8 == 0) ? 0u : 1u);
    mma_tf32_ts_warp(tmem + (uint32_t)nt, al, bh + o, idesc, 1u);
  }
}

// 16 accumulator columns [c0, c0+16) of this thread's row, summed over the K-split pairs: all
// tcgen05.ld of the group are issued before one wait::ld
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void acc_load16(uint32_t tmem, int ew, int c0, int nacc, int slot, float *tot) {
  const uint32_t lane_base = tmem + ((uint32_t)(ew * 32) << 16) + c0;
  uint32_t x0[16], m0[16];
  tmem_ld16_nowait(lane_base, x0);                          // cross terms
  tmem_ld16_nowait(lane_base + (uint32_t)slot, m0);         // main terms, K part 0
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) tot[i] = __uint_as_float(x0[i]) + __uint_as_float(m0[i]);
  for (int q = 1; q < nacc; ++q) {
    tmem_ld16_nowait(lane_base + (uint32_t)((1 + q) * slot), m0);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) tot[i] += __uint_as_float(m0[i]);
  }
}

// Active-column bitmask of a column tile (bit c ⇔ column j0+c has flag 1), computed by one warp
// from flags written by other CTAs in the previous update phase; NT ≤ 128 → 4 words.
__device__ __forceinline__ int tile_mask(const int *flag, int ncol, int lane, uint32_t *mask) {
  int cnt = 0;
#pragma unroll
  for (int w = 0; w < TC_NTMAX / 32; ++w) {
    const int c = w * 32 + lane;
    const int f = (c < ncol) ? (ldv(flag + c) == 1) : 0;
    mask[w] = __ballot_sync(0xffffffffu, f);
    cnt += __popc(mask[w]);
  }
  return cnt;
}
__device__ __forceinline__ int mean_count(const int *flagm, int C, int lane) {
  const int f = (lane < C) ? (ldv(flagm + lane) == 1) : 0;
  return __popc(__ballot_sync(0xffffffffu, f));
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ double2 lds_d2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_d(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a));
  return v;
}

// D(8×8) += A(8×4) · B(4×8) on the FP64 tensor path; lane holds A[lane/4][lane%4], B[lane%4][lane/4]
// and D[lane/4][2·(lane%4) + {0, 1}]
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// fp64 mean-column work of one ring stage, one warp, rows [32·ew, 32·ew + 32) of the tile:
// acc += Φ[rows][k-chunk] · B[k-chunk][C] exactly in fp64 (the staged fp32 Φ tile).  Stage 1 reads
// B from the Dm chunk laid out [c][32], stage 2 from the Um chunk laid out [32][Cp].  Accumulator
// fragment acc[mt][nt] holds rows 32·ew + 8·mt + lane/4, columns 8·nt + 2·(lane%4) + {0, 1}.
// (Measured: the FP64 tensor path beats row-per-thread DFMA here — C3 −10 %, C4 −35 % with DFMA.)
template <bool B_CK, int NTC>
__device__ __forceinline__ void mean_stage(uint32_t a32, uint32_t mb, int ew, int lane, int C, int Cp,
                                           double (&acc)[4][NTC][2]) {
  const int g = lane >> 2, q = lane & 3;
  // all shared-memory operands of the stage first (32 A values, 8·NTC B values per lane), so the
  // FP64 pipe (F2F + DMMA, the binding resource of the mean columns) runs without load gaps
  float af[TK / 4][4];
  double bf[TK / 4][NTC];
#pragma unroll
  for (int ks = 0; ks < TK / 4; ++ks) {
    const int k = 4 * ks + q;
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt) {
      const int n = 8 * nt + g;
      bf[ks][nt] = (n < C) ? lds_d(mb + (uint32_t)(B_CK ? n * TK + k : k * Cp + n) * 8) : 0.0;
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) af[ks][mt] = lds_f32(a32 + sw128_offset(32 * ew + 8 * mt + g, ks) + (uint32_t)q * 4);
  }
#pragma unroll
  for (int ks = 0; ks < TK / 4; ++ks)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const double a = (double)af[ks][mt];
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt) dmma(acc[mt][nt], a, bf[ks][nt]);
    }
}

// tf32 rounding to nearest (ties away from zero, = cvt.rna.tf32.f32 for finite x) on the integer pipe
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// Row r of a staged 128-byte-swizzled fp32 tile (this thread's TMEM lane) as the exact pair
// x = hi + lo, hi = tf32(x), lo = x − hi, written to the TMEM A stage at lane address `ta`: hi in
// columns [0, 32), lo in [32, 64).  The swizzle permutes 16-byte chunks within a row only: logical
// chunk c of row r sits at position c ^ (r & 7), so the 32 lanes of a warp (32 consecutive rows)
// spread each read over all 32 banks.
__device__ __forceinline__ void split_row_tmem32(uint32_t a32, uint32_t ta, int r) {
  // the same with one 32-column store per plane (fewer, larger TMEM writes)
  const uint32_t row = a32 + (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128;
  float hi[32], lo[32];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 v = lds128(row + (uint32_t)((c ^ r) & 7) * 16);
    hi[4 * c + 0] = tf32_rna(v.x); lo[4 * c + 0] = v.x - hi[4 * c + 0];
    hi[4 * c + 1] = tf32_rna(v.y); lo[4 * c + 1] = v.y - hi[4 * c + 1];
    hi[4 * c + 2] = tf32_rna(v.z); lo[4 * c + 2] = v.z - hi[4 * c + 2];
    hi[4 * c + 3] = tf32_rna(v.w); lo[4 * c + 3] = v.w - hi[4 * c + 3];
  }
  tmem_st32(ta, hi);
  tmem_st32(ta + 32, lo);
}
__device__ __forceinline__ void split_row_tmem(uint32_t a32, uint32_t ta, int r) {
  const uint32_t row = a32 + (uint32_t)(r >> 3) * 1024 + (uint32_t)(r & 7) * 128;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float hi[16], lo[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float4 v = lds128(row + (uint32_t)(((4 * h + c) ^ r) & 7) * 16);
      hi[4 * c + 0] = tf32_rna(v.x); lo[4 * c + 0] = v.x - hi[4 * c + 0];
      hi[4 * c + 1] = tf32_rna(v.y); lo[4 * c + 1] = v.y - hi[4 * c + 1];
      hi[4 * c + 2] = tf32_rna(v.z); lo[4 * c + 2] = v.z - hi[4 * c + 2];
      hi[4 * c + 3] = tf32_rna(v.w); lo[4 * c + 3] = v.w - hi[4 * c + 3];
    }
    tmem_st16(ta + 16 * h, hi);
    tmem_st16(ta + 32 + 16 * h, lo);
  }
}

// Per-unit geometry shared by all roles (computed redundantly by every warp).
struct Unit {
  int stage;          // 1 or 2
  int t, ct, rt, sp;
  int ncol;           // columns of the tile (≤ NT)
  int nmma;           // MMA N (0: no probe work)
  bool mean;          // fp64 mean columns ride along
  int nk;             // K chunks
  int k0;             // first K element
  int arow, brow;     // TMA row coordinates of A and B
};

__device__ void report(int *status, int code, int t, int col, int u) {
  if (atomicCAS(status, 0, code) == 0) {
    status[1] = t;
    status[2] = col;
    status[3] = u;
  }
}

// ---- phase 3 -----------------------------------------------------------------------------------
// Alg. 1 lines 3-7 for one probe column by one warp (fp32 vectors, fp64 scalars and dots)
// With `stg` (this warp's 2·D floats of shared memory, when D is small enough: the ring is idle in
// this phase) the first pass also parks d and the new r there, so the direction update re-reads
// shared memory instead of global memory (one dependent global round trip per 256 elements less).
__device__ void update_probe(const KParams &p, int t, int col, int u, int lane, float4 *stg,
                             unsigned long long *tr) {
  if (tr) tr[0] = clock64();
  const Dims &d = p.d;
  const size_t g = (size_t)t * d.P + col;
  float4 *__restrict__ x4 = reinterpret_cast<float4 *>(p.b.X + g * d.D);
  float4 *__restrict__ r4 = reinterpret_cast<float4 *>(p.b.R + g * d.D);
  float4 *__restrict__ d4 = reinterpret_cast<float4 *>(p.b.D32 + g * d.D);
  float4 *__restrict__ dh4 = reinterpret_cast<float4 *>(p.b.Dh + g * d.D);
  float4 *__restrict__ dl4 = reinterpret_cast<float4 *>(p.b.Dl + g * d.D);
  const float4 *__restrict__ w4 = reinterpret_cast<const float4 *>(p.b.W + g * d.D);
  const int n4 = d.D >> 2;
  constexpr int U = 2;   // float4 per lane in flight (per array)
  // the first block of the pass is loaded before the dᵀAd reduction (independent of it: one
  // dependent global round trip less per column)
  float4 dd[U], wv[U], xv[U], rv[U];
#pragma unroll
  for (int v = 0; v < U; ++v) {
    const int i = lane + 32 * v;
    if (i < n4) { dd[v] = ldv(d4 + i); wv[v] = __ldcg(w4 + i); xv[v] = ldv(x4 + i); rv[v] = ldv(r4 + i); }
  }
  // the per-row-tile partials of dᵀAd: one load per lane, then the warp's fixed-order butterfly
  double dpart = 0.0;
  // W and the dᵀAd partials come from other CTAs' stage 2 (acquired through the task counter, no
  // grid barrier): read through L2
  for (int i = lane; i < d.nRT2; i += 32) dpart += __ldcg(p.b.dAd + g * d.nRT2 + i);
  double dAd = warp_sum(dpart);
  const double rr0 = ldv(p.b.rr + g);
  const double rr = (p.dbg_flags & 65536) && !(rr0 > 0.0 && rr0 < 1e300) ? 1.0 : rr0;
  if ((p.dbg_flags & 65536) && !(dAd > 0.0 && dAd < 1e300)) dAd = 1.0;   // diagnostics: timing only
  if (!(dAd > 0.0)) {  // Alg. 1 line 3 breakdown
    if (lane == 0) {
      report(p.b.status, ST_BREAKDOWN, d.t0 + t, col, u + 1);
      p.b.flag[g] = 0;
    }
    return;
  }
  // the step sizes act in fp32 (the vectors' precision; fp32 FMAs: F2F.F64.F32 runs at 2 lanes / clk
  // per SM sub-partition, tools/dmma_test.cu) and the transcript records the values applied
  const float gamf = (float)(rr / dAd);
  const double gam = (double)gamf;
  if (tr) tr[1] = clock64();
  double acc = 0.0;
  for (int i0 = lane; i0 < n4; i0 += 32 * U) {
    if (i0 != lane) {
#pragma unroll
      for (int v = 0; v < U; ++v) {
        const int i = i0 + 32 * v;
        if (i < n4) { dd[v] = ldv(d4 + i); wv[v] = __ldcg(w4 + i); xv[v] = ldv(x4 + i); rv[v] = ldv(r4 + i); }
      }
    }
#pragma unroll
    for (int v = 0; v < U; ++v) {
      const int i = i0 + 32 * v;
      if (i < n4) {
        const float4 dv = dd[v];
        const float4 ad = wv[v];            // Ad from the operator's epilogue
        float4 x = xv[v], r = rv[v];
        x.x = fmaf(gamf, dv.x, x.x);
        x.y = fmaf(gamf, dv.y, x.y);
        x.z = fmaf(gamf, dv.z, x.z);
        x.w = fmaf(gamf, dv.w, x.w);
        r.x = fmaf(-gamf, ad.x, r.x);
        r.y = fmaf(-gamf, ad.y, r.y);
        r.z = fmaf(-gamf, ad.z, r.z);
        r.w = fmaf(-gamf, ad.w, r.w);
        stv(x4 + i, x);
        stv(r4 + i, r);
        if (stg) {
          stg[i] = dv;
          stg[n4 + i] = r;
        }
        acc += (double)fmaf(r.w, r.w, fmaf(r.z, r.z, fmaf(r.y, r.y, r.x * r.x)));   // fp64 across float4s
      }
    }
  }
  if (tr) tr[2] = clock64();
  const double rrn = warp_sum(acc);
  const float xif = (float)(rrn / rr);
  const double xi = (double)xif;
  if (tr) tr[3] = clock64();
  // (timing-only diagnostics: no column retires before the cap, so every variant does the same work)
  const bool conv = !(p.dbg_flags & 65536) && sqrt(rrn) <= p.tol * sqrt((double)d.D);
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
    __syncwarp();
    for (int i0 = lane; i0 < n4; i0 += 32 * U) {
      float4 rv[U], dd[U];
#pragma unroll
      for (int v = 0; v < U; ++v) {
        const int i = i0 + 32 * v;
        if (i < n4) {
          if (stg) { rv[v] = stg[n4 + i]; dd[v] = stg[i]; }   // this lane's own stores: no sync needed
          else { rv[v] = ldv(r4 + i); dd[v] = ldv(d4 + i); }
        }
      }
#pragma unroll
      for (int v = 0; v < U; ++v) {
        const int i = i0 + 32 * v;
        if (i < n4) {
          float4 dv = dd[v];
          dv.x = fmaf(xif, dv.x, rv[v].x);
          dv.y = fmaf(xif, dv.y, rv[v].y);
          dv.z = fmaf(xif, dv.z, rv[v].z);
          dv.w = fmaf(xif, dv.w, rv[v].w);
          stv(d4 + i, dv);
          float4 h4;
          h4.x = tf32_rna(dv.x); h4.y = tf32_rna(dv.y); h4.z = tf32_rna(dv.z); h4.w = tf32_rna(dv.w);
          stv(dh4 + i, h4);
          stv(dl4 + i, make_float4(dv.x - h4.x, dv.y - h4.y, dv.z - h4.z, dv.w - h4.w));
        }
      }
    }
  }
  if (tr) tr[4] = clock64();
}

// the same for one fp64 mean column
__device__ void update_mean(const KParams &p, int t, int c, int u, int lane) {
  const Dims &d = p.d;
  const size_t g = (size_t)t * d.C + c;
  double dpart = 0.0;
  for (int i = lane; i < d.nRT2; i += 32) dpart += __ldcg(p.b.dAdm + g * d.nRT2 + i);
  double dAd = warp_sum(dpart);
  double rr = ldv(p.b.rrm + g);
  if (p.dbg_flags & 65536) {   // diagnostics: timing only
    if (!(rr > 0.0 && rr < 1e300)) rr = 1.0;
    if (!(dAd > 0.0 && dAd < 1e300)) dAd = 1.0;
  }
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
  constexpr int U = 2;
  for (int i0 = lane; i0 < n2; i0 += 32 * U) {
    double2 dd[U], ww[U], xx[U], rn[U];
#pragma unroll
    for (int v = 0; v < U; ++v) {
      const int i = i0 + 32 * v;
      if (i < n2) { dd[v] = ldv(dv + i); ww[v] = __ldcg(w + i); xx[v] = ldv(x + i); rn[v] = ldv(r + i); }
    }
#pragma unroll
    for (int v = 0; v < U; ++v) {
      const int i = i0 + 32 * v;
      if (i < n2) {
        const double adx = ww[v].x, ady = ww[v].y;
        xx[v].x = fma(gam, dd[v].x, xx[v].x);
        xx[v].y = fma(gam, dd[v].y, xx[v].y);
        rn[v].x = fma(-gam, adx, rn[v].x);
        rn[v].y = fma(-gam, ady, rn[v].y);
        stv(x + i, xx[v]);
        stv(r + i, rn[v]);
        acc = fma(rn[v].x, rn[v].x, acc);
        acc = fma(rn[v].y, rn[v].y, acc);
      }
    }
  }
  const double rrn = warp_sum(acc);
  const double xi = rrn / rr;
  const bool conv = !(p.dbg_flags & 65536) && sqrt(rrn) <= p.tol_mean * sqrt(p.b.bnorm2[t]);
  const bool stop = conv || (u + 1 >= d.cap);
  if (lane == 0) {
    p.b.stepsm[g] = u + 1;
    p.b.rrm[g] = rrn;
    if (stop) p.b.flagm[g] = conv ? 0 : 2;
    else atomicAdd(p.b.alive + u, 1);
  }
  if (!stop) {
    __syncwarp();
    for (int i0 = lane; i0 < n2; i0 += 32 * U) {
      double2 rn[U], dd[U];
#pragma unroll
      for (int v = 0; v < U; ++v) {
        const int i = i0 + 32 * v;
        if (i < n2) { rn[v] = ldv(r + i); dd[v] = ldv(dv + i); }
      }
#pragma unroll
      for (int v = 0; v < U; ++v) {
        const int i = i0 + 32 * v;
        if (i < n2) {
          dd[v].x = fma(xi, dd[v].x, rn[v].x);
          dd[v].y = fma(xi, dd[v].y, rn[v].y);
          stv(dv + i, dd[v]);
        }
      }
    }
  }
}

// ---- unit geometry ---------------------------------------------------------------------------
// Shared Φ: the units of a phase form one large GEMM (rows of Φ/Φᵀ × all tasks' columns).  Units
// are rasterised in bands of RB row tiles: inside a band the row tile varies fastest, then the
// column tile, then the task, so a wave of ~148 concurrent units reads RB row tiles of Φ and
// ~148 / RB column tiles of the tasks' operands at each K step (L2 reuse of both operands).
constexpr int RB = 8;
__device__ __forceinline__ void decode_banded(int w, int Tl, int nCT, int nRT, int *t, int *ct, int *rt) {
  const int full = nRT / RB;                       // complete bands
  const int per_band = Tl * nCT * RB;
  int band = w / per_band, rb = RB;
  int r = w - band * per_band;
  if (band >= full) {                              // the last, partial band
    band = full;
    rb = nRT - full * RB;
    r = w - full * per_band;
  }
  *rt = band * RB + r % rb;
  r /= rb;
  *ct = r % nCT;
  *t = r / nCT;
}

// Column tile of unit w when the column tiles of a row tile sit on neighbouring CTAs: rotated by
// the round k = w / G so that a CTA alternates between column tiles (the fp64 mean columns ride
// with column tile 0: without the rotation, G being a multiple of the group, every CTA would see
// the same column tile in every round — all the mean work on half of the CTAs).  A bijection
// whenever the group (the nCT consecutive units sharing everything but ct) never straddles a
// round boundary, i.e. G % group == 0.
__device__ __forceinline__ int rotate_ct(int c, int w, int G, int group, int nCT) {
  return (G % group == 0) ? (c + w / G) % nCT : c;
}

// Units are dealt to G dealers (CTAs, or CTA pairs: then a unit covers the row-tile pair (2ρ, 2ρ+1)
// and rank r of the pair takes row tile 2ρ + r; nRTu = the phase's row tiles or row-tile pairs)
__device__ __forceinline__ int nrt_units(int nrt, int pair) { return pair ? (nrt + 1) / 2 : nrt; }
__device__ __forceinline__ Unit make_unit1(const Dims &d, const TcCfg &tc, int w, int G, int rank) {
  Unit x;
  x.stage = 1;
  const int nRTu = nrt_units(d.nRT1, tc.pair);
  if (d.shared_phi) {
    x.sp = w % d.S1;
    decode_banded(w / d.S1, d.Tl, d.nCT, nRTu, &x.t, &x.ct, &x.rt);
  } else {
    // column tiles of a row tile on neighbouring CTAs: they stream the same Φ rows together (L2)
    x.sp = w % d.S1;
    int r = w / d.S1;
    x.ct = rotate_ct(r % d.nCT, w, G, d.S1 * d.nCT, d.nCT);
    r /= d.nCT;
    x.rt = r % nRTu;
    x.t = r / nRTu;
  }
  if (tc.pair) x.rt = 2 * x.rt + rank;
  const int j0 = x.ct * tc.NT;
  x.ncol = min(tc.NT, d.P - j0);
  x.k0 = x.sp * d.K1;
  const int ke = min(d.D, x.k0 + d.K1);
  x.nk = (ke - x.k0 + TK - 1) / TK;
  x.arow = x.rt * TM;                              // row of Φ_t (per-task maps)
  x.brow = j0;                                     // first direction column of the tile
  return x;
}
__device__ __forceinline__ Unit make_unit2(const Dims &d, const TcCfg &tc, int w, int G, int rank) {
  Unit x;
  x.stage = 2;
  x.sp = 0;
  const int nRTu = nrt_units(d.nRT2, tc.pair);
  if (d.shared_phi) {
    decode_banded(w, d.Tl, d.nCT, nRTu, &x.t, &x.ct, &x.rt);
  } else {
    x.ct = rotate_ct(w % d.nCT, w, G, d.nCT, d.nCT);
    const int r = w / d.nCT;
    x.rt = r % nRTu;
    x.t = r / nRTu;
  }
  if (tc.pair) x.rt = 2 * x.rt + rank;
  const int j0 = x.ct * tc.NT;
  x.ncol = min(tc.NT, d.P - j0);
  x.k0 = 0;
  x.nk = (d.N + TK - 1) / TK;
  x.arow = x.rt * TM;                              // row of Φ_tᵀ
  x.brow = j0;
  return x;
}

// which work the unit has (every warp evaluates it from the same settled flags)
__device__ __forceinline__ void unit_work(const KParams &p, Unit &x, int lane, uint32_t *mask) {
  const Dims &d = p.d;
  const int j0 = x.ct * p.tc.NT;
  const int m = tile_mask(p.b.flag + (size_t)x.t * d.P + j0, x.ncol, lane, mask);
  // a pair's MMA spans the whole tile (each CTA stages NT/2 columns; padding columns are zero-filled)
  x.nmma = m ? (p.tc.pair ? p.tc.NT : ((x.ncol + 15) & ~15)) : 0;
  x.mean = x.ct == 0 && !(p.dbg_flags & 512) && mean_count(p.b.flagm + (size_t)x.t * d.C, d.C, lane) > 0;
}

// ring: chunk G lives in stage G % S; full / empty phase of chunk G is G / S.  The TMEM A ring
// (SA stages) counts the chunks with probe MMAs the same way (afull / aempty).
struct RingCtl {
  int S;
  uint32_t g;      // chunks handled so far by this role
  int st;          // = g % S (kept incrementally: no integer division in the K loops)
  uint32_t ph;     // = (g / S) & 1
  __device__ __forceinline__ void next() {
    ++g;
    if (++st == S) { st = 0; ph ^= 1u; }
  }
  int SA;
  uint32_t ag;     // TMEM A stages handled so far (A warps, MMA warp)
  int ast;         // = ag % SA
  uint32_t aph;    // = (ag / SA) & 1
  __device__ __forceinline__ void nexta() {
    ++ag;
    if (++ast == SA) { ast = 0; aph ^= 1u; }
  }
  uint32_t ti;     // accumulator tiles handled so far
  uint32_t tf[2];  // tiles committed to / drained from each TMEM accumulator buffer (tfull phases)
  uint32_t te[2];  // MMA warp: tempty completions expected per buffer (a single-buffered tile in the
                   // double-buffer layout spans both buffers and is released on both)
  uint32_t di;     // stage-2 d tiles handled so far (dfull / dempty phases)
  uint32_t smean;  // producer: bit s = the chunk last placed in slot s belongs to a mean unit
  uint32_t mcnt[MAXST];  // producer: mean chunks placed in each slot (mdone phases)
};

// ---- producer (warp 0, converged; one elected lane issues) ---------------------------------------------------------------
template <bool PR>
__device__ __forceinline__ void produce(const KParams &p, const TcMaps &mp, unsigned char *sm, PSmemTail &tl,
                                        RingCtl &rc, const Unit &x, unsigned long long *tr, uint32_t rank) {
  if (tr && (threadIdx.x & 31) == 0) tr[84] = clock64();
  const uint32_t b_bytes = (uint32_t)p.tc.NT * 128;       // one plane (hi or lo) of the tile's B
  const uint32_t mean_tx = x.stage == 1 ? (uint32_t)p.d.C * TK * 8 : (uint32_t)TK * p.d.Cp * 8;
  // the local full barrier counts the A tile and mean chunk (and B when unpaired); a pair's B halves
  // (hi | lo planes of NT/2 rows each per CTA) count on the leader's bfull
  const uint32_t bytes = A_BYTES + ((x.nmma && !PR) ? 2 * b_bytes : 0) + (x.mean ? mean_tx : 0);
  const uint32_t b_stage = PR ? b_bytes : 2 * b_bytes;    // B bytes in this CTA's stage
  for (int kc = 0; kc < x.nk; ++kc) {
    const uint32_t G = rc.g;
    const int st = rc.st;
    const uint32_t cph = rc.ph;
    rc.next();
    if (G >= (uint32_t)rc.S) {
      mbar_wait(&tl.empty[st], cph ^ 1u);     // chunk G − S (same slot): MMAs and split done
      if ((rc.smean >> st) & 1u) mbar_wait(&tl.mdone[st], (rc.mcnt[st] - 1) & 1);   // its fp64 work too
    }
    if (x.mean) {
      rc.smean |= 1u << st;
      rc.mcnt[st]++;
    } else {
      rc.smean &= ~(1u << st);
    }
    if (tr && kc < 16 && (threadIdx.x & 31) == 0) tr[kc] = clock64();
    unsigned char *base = sm + (size_t)st * p.tc.stage_bytes;
    uint64_t *fb = &tl.full[st];
    if (p.dbg_flags & 128) {                  // diagnostic: no operand traffic
      if ((threadIdx.x & 31) == 0) {
        mbar_arrive(fb);
        if (PR && x.nmma && rank == 0) mbar_arrive(&tl.bfull[st]);
      }
      continue;
    }
    mbar_arrive_expect_tx_warp(fb, bytes);
    const int k = x.k0 + kc * TK;
    // stage layout: fp32 A tile | B hi | B lo | fp64 mean-column chunk
    // every operand map is per task ([task][rows][cols]): a box never reaches into the next task's
    // rows (out-of-range rows and K columns are zero-filled), so tasks are isolated even where a tile
    // or a K chunk overhangs the task's matrix
    const int at = p.d.shared_phi ? 0 : x.t;
    if (p.tc.pf && (threadIdx.x & 31) == 0) {   // A tiles PF chunks ahead into L2
      const CUtensorMap *am = x.stage == 1 ? &mp.phi : &mp.phit;
      for (int k2 = (kc == 0 ? rc.S : kc + p.tc.pf); k2 <= kc + p.tc.pf && k2 < x.nk; ++k2)
        tma_prefetch_3d(am, x.k0 + k2 * TK, x.arow, at);
    }
    const CUtensorMap *bmap = x.stage == 1 ? &mp.d_hl : &mp.u_hl;
    if (PR && x.nmma) {
      const uint32_t bl = mapa_shared(smem_u32(&tl.bfull[st]), 0);
      if (rank == 0) mbar_arrive_expect_tx_warp(&tl.bfull[st], 2 * b_bytes);
      tma_load_4d_warp_pair(base + A_BYTES, bmap, k, x.brow + (int)rank * (p.tc.NT / 2), x.t, 0, bl);
    }
    if (p.tc.l2hint) {
      // A streams (evict first); B and the mean chunk are re-read by the task's other row tiles
      const uint64_t pa = l2_policy_evict_first(), pb = l2_policy_evict_last();
      tma_load_3d_warp_hint(base, x.stage == 1 ? &mp.phi : &mp.phit, k, x.arow, at, fb, pa);
      if (x.nmma && !PR) tma_load_4d_warp_hint(base + A_BYTES, bmap, k, x.brow, x.t, 0, fb, pb);
      if (x.mean) {
        if (x.stage == 1) tma_load_3d_warp_hint(base + A_BYTES + b_stage, &mp.dm, k, 0, x.t, fb, pb);
        else tma_load_3d_warp_hint(base + A_BYTES + b_stage, &mp.um, 0, k, x.t, fb, pb);
      }
    } else if (x.stage == 1) {
      tma_load_3d_warp(base, &mp.phi, k, x.arow, at, fb);
      if (x.nmma && !PR) tma_load_4d_warp(base + A_BYTES, bmap, k, x.brow, x.t, 0, fb);   // hi | lo tiles
      if (x.mean) tma_load_3d_warp(base + A_BYTES + b_stage, &mp.dm, k, 0, x.t, fb);
    } else {
      tma_load_3d_warp(base, &mp.phit, k, x.arow, at, fb);
      if (x.nmma && !PR) tma_load_4d_warp(base + A_BYTES, bmap, k, x.brow, x.t, 0, fb);
      if (x.mean) tma_load_3d_warp(base + A_BYTES + b_stage, &mp.um, 0, k, x.t, fb);
    }
    if (tr && kc < 16 && (threadIdx.x & 31) == 0) tr[16 + kc] = clock64();
  }
  if (x.stage == 2 && x.nmma && p.tc.use_dtile) {
    // the epilogue's d tile (rows d0..d0+127 of the tile's NT direction columns), after the K loop
    // so the ring keeps streaming while the previous tile's epilogue still reads its d tile
    if (rc.di > 0) mbar_wait(&tl.dempty, (rc.di - 1) & 1);
    unsigned char *dt = sm + (size_t)rc.S * p.tc.stage_bytes;
    if (p.dbg_flags & 128) {
      if ((threadIdx.x & 31) == 0) mbar_arrive(&tl.dfull);
    } else {
      mbar_arrive_expect_tx_warp(&tl.dfull, p.tc.dtile_bytes);
      tma_load_3d_warp(dt, &mp.d32, x.rt * TM, x.ct * p.tc.NT, x.t, &tl.dfull);
    }
    rc.di++;
  }
}

// ---- MMA issuer (warp 1, converged; one elected lane issues) ------------------------------------
// (CTA pairs: run by the leader's MMA warp only; its commits arrive on both CTAs' barriers)
template <bool PR>
__device__ __forceinline__ void mma_unit(const KParams &p, unsigned char *sm, PSmemTail &tl, RingCtl &rc,
                                         uint32_t tmem, const Unit &x, unsigned long long *tr, uint32_t rank) {
  const TcCfg &tc = p.tc;
  const int lane = threadIdx.x & 31;
  if (PR && rank != 0) {
    // a pair's peer: the leader issues the MMAs (and its commits release this CTA's stages); this
    // warp only keeps its ring position and releases its slots of mean-only units (see below)
    for (int kc = 0; kc < x.nk; ++kc) {
      const int st = rc.st;
      const uint32_t ph = rc.ph;
      rc.next();
      if (!x.nmma) {
        mbar_wait(&tl.full[st], ph);
        if (lane == 0) mbar_arrive(&tl.empty[st]);
      }
      __syncwarp();
    }
    return;
  }
  const uint32_t lo_off = (uint32_t)tc.NT * 128 / (PR ? 2 : 1);
  const int nacc = unit_nacc(tc, x.nk, p.dbg_flags);
  const uint32_t idesc = idesc_tf32(PR ? 2 * TM : TM, x.nmma > 0 ? x.nmma : 32);
  const bool dbl = unit_dbl(tc, x.nk, p.dbg_flags);
  // a full double-buffered tile: the 2-MMA form (N = 2·NT ≤ 256; unpaired only: a pair's stage
  // holds half of the hi and of the lo plane, not a contiguous [hi | lo])
  const bool cat = !PR && dbl && x.nmma == tc.NT && tc.slot == tc.NT && 2 * tc.NT <= 256 && !(p.dbg_flags & 4096);
  const uint32_t idesc2 = idesc_tf32(TM, cat ? 2 * tc.NT : 16);
  const int bi = dbl ? (int)(rc.ti & 1) : 0;
  const uint32_t tacc = tmem + (uint32_t)(bi * 2 * tc.slot);
  if (x.nmma) {
    // the epilogue has drained this buffer's previous tile (both buffers for a 512-column tile)
    if (rc.te[bi] > 0) mbar_wait(&tl.tempty[bi], (rc.te[bi] - 1) & 1);
    if (!dbl && rc.te[1] > 0) mbar_wait(&tl.tempty[1], (rc.te[1] - 1) & 1);
    fence_after_sync();
  }
  for (int kc = 0; kc < x.nk; ++kc) {
    const int st = rc.st;
    const uint32_t ph = rc.ph;
    rc.next();
    if (x.nmma) {
      const int sa = rc.ast;
      mbar_wait(&tl.afull[sa], rc.aph);       // A stage written (the A warps waited full[st] first)
      rc.nexta();
      mbar_wait(PR ? &tl.bfull[st] : &tl.full[st], ph);   // B staged (a pair: both halves)
      if (tr && kc < 16 && lane == 0) tr[32 + kc] = clock64();
      if (!(p.dbg_flags & 2)) {
        fence_after_sync();
        const int q = (kc * nacc) / x.nk;
        const int qfirst = (q * x.nk + nacc - 1) / nacc;
        if (cat)
          mma_stage_cat(tacc, tmem + (uint32_t)(tc.acol0 + 64 * sa), sm + (size_t)st * tc.stage_bytes, idesc2, idesc,
                        tc.NT, kc == 0);
        else
          mma_stage<PR>(tacc, tmem + (uint32_t)(tc.acol0 + 64 * sa), sm + (size_t)st * tc.stage_bytes, lo_off, idesc,
                        q, tc.slot, kc == qfirst, kc == 0);
        if (PR) {
          mma_commit_warp_pair(&tl.aempty[sa]);   // both CTAs: the MMAs have read their A stages
          mma_commit_warp_pair(&tl.empty[st]);    // ... and their B halves
        } else {
          mma_commit_warp(&tl.aempty[sa]);      // the MMAs have read the A stage
          mma_commit_warp(&tl.empty[st]);       // ... and the B tiles
        }
      } else if (lane == 0) {
        mbar_arrive(&tl.aempty[sa]);
        mbar_arrive(&tl.empty[st]);
        if (PR) {
          mbar_arrive_cluster(mapa_shared(smem_u32(&tl.aempty[sa]), 1));
          mbar_arrive_cluster(mapa_shared(smem_u32(&tl.empty[st]), 1));
        }
      }
    } else {
      // no probe work in this unit (mean columns only): the MMA warp's share of empty[st] — after
      // full[st], so it never runs ahead of the ring (an arrival for chunk G + S landing in chunk G's
      // phase would complete that phase early and shift every later one: a hang).  A pair's CTAs
      // each release their own slot here (the peer's MMA warp runs this path too).
      mbar_wait(&tl.full[st], ph);
      if (lane == 0) mbar_arrive(&tl.empty[st]);
    }
    __syncwarp();
  }
  if (x.nmma) {
    if (p.dbg_flags & 2) {
      if (lane == 0) {
        mbar_arrive(&tl.tfull[bi]);
        if (PR) mbar_arrive_cluster(mapa_shared(smem_u32(&tl.tfull[bi]), 1));
      }
    } else if (PR) {
      mma_commit_warp_pair(&tl.tfull[bi]);   // both CTAs' accumulators ready
    } else {
      mma_commit_warp(&tl.tfull[bi]);        // all MMAs of the tile complete → accumulator ready
    }
    rc.tf[bi]++;
    rc.te[bi]++;
    if (!dbl && tc.dbl) rc.te[1]++;          // the tile also covers buffer 1's columns
    rc.ti++;
  }
}

// named barrier 2: the epilogue warps (6-9)

// Split-K handoff of a stage-1 tile (S1 > 1), called by the epilogue warps once this CTA's partial
// tiles (probe and mean columns) are written; returns the rows [rb, re) of the tile
// this CTA sums over the S1 partials, in split order (deterministic):
//  * cooperative (all stage-1 units co-resident, small configs): every split CTA waits on the tile
//    counter for all S1 partials and reduces its 1/S1 share of the rows;
//  * last arriver (several units per CTA): the CTA that completes the tile's S1 arrivals of this
//    step reduces the whole tile, the others move on.
// The tile counters only grow (S1 arrivals per active tile and step, zeroed at init).
__device__ __forceinline__ void split_handoff(const KParams &p, const Unit &x, PSmemTail &tl, int *rb, int *re) {
  const Dims &d = p.d;
  // the epilogue warps' partial stores are ordered before EPI0's release by the barrier (a
  // gpu-scope release is cumulative over what the releasing thread has observed)
  epi_sync();
  int *cnt = p.b.tilecnt + ((size_t)x.t * d.nCT + x.ct) * d.nRT1 + x.rt;
  if (threadIdx.x == EPI0) {
    int ticket;
    asm volatile("atom.add.release.gpu.global.s32 %0, [%1], 1;\n" : "=r"(ticket) : "l"(cnt) : "memory");
    if (d.split_coop) {
      const int target = (ticket / d.S1 + 1) * d.S1;
      int v;
      do {
        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(cnt) : "memory");
      } while (v < target);
    }
    tl.last = (ticket % d.S1) == d.S1 - 1;
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  }
  epi_sync();
  const int n0 = x.rt * TM, rows = min(TM, d.N - n0);
  if (d.split_coop) {
    const int rs = ((rows + d.S1 - 1) / d.S1 + 3) & ~3;     // rows per share (×4: float4 rows)
    *rb = min(rows, x.sp * rs);
    *re = min(rows, *rb + rs);
  } else {
    *rb = 0;
    *re = tl.last ? rows : 0;
  }
}

// ---- A warps (2-5): the TMEM A stages ------------------------------------------------------------
template <bool PR>
__device__ void a_unit(const KParams &p, unsigned char *sm, PSmemTail &tl, RingCtl &rc, uint32_t tmem, const Unit &x,
                       unsigned long long *tr, unsigned long long *tr4) {
  const TcCfg &tc = p.tc;
  const int aq = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;   // TMEM lane quarter of this warp
  const uint32_t ta_lane = tmem + ((uint32_t)(32 * aq) << 16) + (uint32_t)tc.acol0;
  for (int kc = 0; kc < x.nk; ++kc) {
    const int st = rc.st;
    mbar_wait(&tl.full[st], rc.ph);
    rc.next();
    if (tr && kc < 16) tr[48 + kc] = clock64();
    if (x.nmma) {
      const uint32_t base = smem_u32(sm) + (uint32_t)st * tc.stage_bytes;
      const int sa = rc.ast;
      if (rc.ag >= (uint32_t)rc.SA) mbar_wait(&tl.aempty[sa], rc.aph ^ 1u);   // MMAs of chunk − SA done
      rc.nexta();
      if (tr && kc < 16) tr[64 + kc] = clock64();
      fence_after_sync();
      if (p.dbg_flags & (131072 | 262144)) {
        // diagnostics (timing only): 131072 split constants into TMEM (no smem reads), 262144 read and
        // split the tile but do not store it to TMEM (a value sink keeps the work)
        if (p.dbg_flags & 131072) {
          float z[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) z[i] = (float)i;
          const uint32_t ta = ta_lane + (uint32_t)(64 * sa);
          tmem_st16(ta, z); tmem_st16(ta + 16, z); tmem_st16(ta + 32, z); tmem_st16(ta + 48, z);
        } else {
          const uint32_t row = base + (uint32_t)((32 * aq + lane) >> 3) * 1024 + (uint32_t)((32 * aq + lane) & 7) * 128;
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = lds128(row + (uint32_t)((c ^ lane) & 7) * 16);
            acc += (v.x - tf32_rna(v.x)) + (v.y - tf32_rna(v.y)) + (v.z - tf32_rna(v.z)) + (v.w - tf32_rna(v.w));
          }
          if (acc == 1.2345e-30f) p.b.status[7] = 1;
        }
      } else if (p.dbg_flags & 524288) {
        split_row_tmem32(base, ta_lane + (uint32_t)(64 * sa), 32 * aq + lane);
      } else if (!(p.dbg_flags & 4)) split_row_tmem(base, ta_lane + (uint32_t)(64 * sa), 32 * aq + lane);
      tmem_wait_st();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) {   // a pair's leader issues the MMA: its afull counts both CTAs' A warps
        if (PR) mbar_arrive_cluster(mapa_shared(smem_u32(&tl.afull[sa]), 0));
        else mbar_arrive(&tl.afull[sa]);
      }
      if (tr && kc < 16) tr[90 + kc] = clock64();
      if (tr4 && lane == 0 && kc < 16) tr4[16 * aq + kc] = clock64();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&tl.empty[st]);
    if (tr && kc < 14) tr[106 + kc] = clock64();
  }
}

// ---- epilogue warps, K loop of a unit: the fp64 mean columns on the FP64 tensor path -----------
// Only chunks of mean units are waited for and released (mdone; the producer refills a slot that
// held a mean chunk only after mdone, so full's phase parity cannot alias); the ring position still
// advances over every chunk.
template <int NTC>
__device__ __forceinline__ void mean_kloop(const KParams &p, unsigned char *sm, PSmemTail &tl, RingCtl &rc,
                                           const Unit &x, double (&macc)[4][NTC][2], unsigned long long *trm) {
  const TcCfg &tc = p.tc;
  const int ew = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;
  const uint32_t mu_off = A_BYTES + (tc.pair ? 1u : 2u) * (uint32_t)tc.NT * 128;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt) macc[mt][nt][0] = macc[mt][nt][1] = 0.0;
  for (int kc = 0; kc < x.nk; ++kc) {
    const int st = rc.st;
    const uint32_t ph = rc.ph;
    rc.next();
    if (x.mean) {
      mbar_wait(&tl.full[st], ph);
      if (trm && threadIdx.x == EPI0 && kc < 16) trm[16 + kc] = clock64();
      if (!(p.dbg_flags & 1)) {
        const uint32_t base = smem_u32(sm) + (uint32_t)st * tc.stage_bytes;
        if (x.stage == 1) mean_stage<true, NTC>(base, base + mu_off, ew, lane, p.d.C, p.d.Cp, macc);
        else mean_stage<false, NTC>(base, base + mu_off, ew, lane, p.d.C, p.d.Cp, macc);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tl.mdone[st]);
      if (trm && threadIdx.x == EPI0 && kc < 16) trm[kc] = clock64();
    }
  }
}

// ---- epilogue warps (6-9): a unit's fp64 mean columns and its probe accumulator tile ----------
// TMEM accumulator buffer of a tile: two buffers (columns [0, 2·slot) and [2·slot, 4·slot)) when
// double-buffered, so the MMA warp starts the next tile while this one drains
__device__ __forceinline__ int acc_buf(const RingCtl &rc, bool dbl) { return dbl ? (int)(rc.ti & 1) : 0; }

// Stage-2 epilogue, column groups [c0, c0 + 16) of the tile: W = β·acc + α_c ⊙ d for row dd of
// this thread (its TMEM lane), W stored, fp64 partial dᵀW per column reduced over the warp's 32
// rows into tl.red[warp % 4]; d from the smem d tile.  (Measured: sharing the drain of a CTA's
// last tile with the A warps does not pay — they join only after their own mean epilogue.)
template <int CC>
__device__ __forceinline__ void drain2_groups(const KParams &p, PSmemTail &tl, const Unit &x, uint32_t tacc,
                                              int nacc, const float *dtile, const float (&alpha)[CC], int g0,
                                              int gstep) {
  const Dims &d = p.d;
  const TcCfg &tc = p.tc;
  const int ew = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31, r = 32 * ew + lane;
  const int D = d.D, C = d.C;
  const int j0 = x.ct * tc.NT;
  const int dd = x.rt * TM + r;
  const bool rv = dd < D;
  const float betaf = (float)p.beta;
  const float *__restrict__ arow = p.b.alpha32 + dd;
  float *__restrict__ Wc = p.b.W + ((size_t)x.t * d.P + j0) * D + dd;
  for (int c0 = 16 * g0; c0 < x.nmma; c0 += 16 * gstep) {
    float dv[16], tot[16], a[16], w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) dv[i] = rv ? dtile[(c0 + i) * TM + r] : 0.f;
    acc_load16(tacc, ew, c0, nacc, tc.slot, tot);
    // α_c of this row, c = cluster of column j0 + c0 + i
    const int jc = j0 + c0, cl0 = jc / d.K;
    if (d.K >= 16) {   // ≤ 2 clusters in a group: column i in cluster cl0 while i < nb (α preloaded)
      const int nb = (cl0 + 1) * d.K - jc;
      float a0 = alpha[0], a1 = alpha[0];
#pragma unroll
      for (int c = 1; c < CC; ++c) {
        if (c == cl0) a0 = alpha[c];
        if (c == cl0 + 1) a1 = alpha[c];
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = i < nb ? a0 : a1;
    } else {
      int cl = cl0, rem = jc - cl0 * d.K;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        a[i] = rv ? __ldg(arow + (size_t)min(cl, C - 1) * D) : 0.f;
        if (++rem == d.K) { rem = 0; ++cl; }
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = fmaf(betaf, tot[i], a[i] * dv[i]);
    if (rv) {   // columns of retired probes get a W too (never read); MMA padding past ncol is not stored
      float *wc = Wc + (uint32_t)c0 * (uint32_t)D;
      const int nv = x.ncol - c0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < nv) *wc = w[i];
        wc += D;
      }
    }
    float dp[16], de[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      dp[i] = dv[i] * w[i];
      de[i] = fmaf(dv[i], w[i], -dp[i]);
    }
    int idx;
    const double sum = warp_reduce16_f(dp, de, lane, &idx);
    if ((lane & 1) == 0) tl.red[ew][c0 + idx] = sum;
  }
}

// A warps: the odd column groups of a CTA's last stage-2 tile of the phase, and of every long
// stage-2 tile carrying fp64 mean columns (help_mean), while the epilogue warps take the even
// groups after their fp64 mean work.  A long mean unit's pace is the epilogue warps' (DMMA K loop
// ≈ 1.4-1.7k clk per chunk against ≈ 0.5k of tcgen05 MMAs, then the drain), so the A warps, idle
// for most of it, halve the drain; on short units (C2: 8 chunks) the MMA warp would stall on the
// next unit's splits instead (measured C3 +1.9 %, C2 −0.5 % when applied to all mean units).
__device__ __forceinline__ bool help_mean(const KParams &p, const Unit &x) {
  return x.mean && x.nk >= 16 && !(p.dbg_flags & 16384);
}
template <int CC>
__device__ void a_help_drain2(const KParams &p, unsigned char *sm, PSmemTail &tl, const RingCtl &rc, const Unit &x) {
  const Dims &d = p.d;
  const TcCfg &tc = p.tc;
  float alpha[CC];
  const int dd = x.rt * TM + 32 * ((threadIdx.x >> 5) & 3) + (threadIdx.x & 31);
#pragma unroll
  for (int c = 0; c < CC; ++c) alpha[c] = (c < d.C && dd < d.D) ? __ldg(p.b.alpha32 + (size_t)c * d.D + dd) : 0.f;
  pair_sync();
  // the epilogue waited on tfull; this barrier plus the fence orders these warps' tcgen05.ld after
  // the MMAs' completion (tcgen05 memory model: thread sync, then fence::after_thread_sync)
  fence_after_sync();
  drain2_groups<CC>(p, tl, x, tl.help_tacc, unit_nacc(tc, x.nk, p.dbg_flags),
                    reinterpret_cast<const float *>(sm + (size_t)rc.S * tc.stage_bytes), alpha, 1, 2);
  fence_before_sync();                        // these tcgen05.ld before the epilogue's tempty release
  pair_sync();                                // W stores ordered before the epilogue's completion release
}

// the accumulator buffer drained: the MMA warp (a pair's leader) may overwrite it
template <bool PR>
__device__ __forceinline__ void tempty_arrive(PSmemTail &tl, int bi, bool both) {
  if (PR) {
    mbar_arrive_cluster(mapa_shared(smem_u32(&tl.tempty[bi]), 0));
    if (both) mbar_arrive_cluster(mapa_shared(smem_u32(&tl.tempty[1]), 0));
  } else {
    mbar_arrive(&tl.tempty[bi]);
    if (both) mbar_arrive(&tl.tempty[1]);
  }
}

template <int CC, bool PR>
__device__ void probe_epilogue(const KParams &p, unsigned char *sm, PSmemTail &tl, RingCtl &rc, uint32_t tmem,
                               const Unit &x, const uint32_t *mask_in, unsigned long long *tr, bool helped) {
  if (tr && threadIdx.x != EPI0) tr = nullptr;
  const Dims &d = p.d;
  const TcCfg &tc = p.tc;
  const int et = threadIdx.x - EPI0, ew = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;
  const int r = 32 * ew + lane;              // tile row = TMEM lane (warp w reads lanes 32·(w % 4) + ...)
  const int N = d.N, D = d.D, P = d.P, C = d.C;
  const int nacc = unit_nacc(tc, x.nk, p.dbg_flags);
  const bool dbl = unit_dbl(tc, x.nk, p.dbg_flags);
  const int j0 = x.ct * tc.NT;
  if (lane < TC_NTMAX / 32) {
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < TC_NTMAX / 32; ++i)
      if (i == lane) v = mask_in[i];
    tl.emask[ew][lane] = v;
  }
  __syncwarp();
  const uint32_t *mask = tl.emask[ew];
  // the fp64 mean columns' share of the K loop (DMMA on the staged tiles, beside the A warps' split)
  constexpr int NTC = (CC + 7) / 8;
  double macc[4][NTC][2];
  mean_kloop<NTC>(p, sm, tl, rc, x, macc, tr ? tr + 224 : nullptr);
  const int fg = lane >> 2, fq = lane & 3;   // DMMA fragment row group / column pair of this lane
  if (x.stage == 1 && x.mean) {              // Um = Φ·Dm rows of this tile (or this split's partial)
    double *dst = d.S1 == 1 ? p.b.Um + (size_t)x.t * N * d.Cp : p.b.Umpart + ((size_t)x.t * d.S1 + x.sp) * N * d.Cp;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int nn = x.rt * TM + 32 * ew + 8 * mt + fg;
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt) {
        const int c = 8 * nt + 2 * fq;         // Cp is even: columns c, c+1 are both < Cp or both ≥ C
        if (nn < N && c < C)
          stv(reinterpret_cast<double2 *>(dst + (size_t)nn * d.Cp + c), make_double2(macc[mt][nt][0], macc[mt][nt][1]));
      }
    }
  }
  if (x.stage == 2 && x.mean) {
    // Wm = β·acc + α ⊙ dm on this lane's fragment rows / columns, and the partial dᵀWm per column
    // over the tile (fragment rows, the 8 row groups of the warp, then the 4 warps)
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * nt + 2 * fq + e;
        double dot = 0.0;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const int de = x.rt * TM + 32 * ew + 8 * mt + fg;
          if (c < C && de < D) {
            const size_t o = ((size_t)x.t * C + c) * D + de;
            const double dmv = ldv(p.b.Dm + o);
            const double wv = fma(p.beta, macc[mt][nt][e], p.b.alpha64[(size_t)c * D + de] * dmv);
            stv(p.b.Wm + o, wv);
            dot = fma(dmv, wv, dot);
          }
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (fg == 0 && c < C) tl.redm[ew][c] = dot;
      }
    }
    epi_sync();
    if (et < C && x.rt < d.nRT2)
      stv(p.b.dAdm + ((size_t)x.t * C + et) * d.nRT2 + x.rt, tl.redm[0][et] + tl.redm[1][et] + tl.redm[2][et] + tl.redm[3][et]);
    epi_sync();                               // tl.redm is reused by the next unit
  }
  uint32_t tacc = tmem;                      // this tile's accumulator buffer
  // stage 2: α_c of this thread's row for every cluster (read-only during the E-step: the
  // non-coherent path), loaded while the accumulator is still being computed
  float alpha[CC];
  {
    const int dd = x.rt * TM + 32 * ew + lane;
#pragma unroll
    for (int c = 0; c < CC; ++c)
      alpha[c] = (x.stage == 2 && c < C && dd < D) ? __ldg(p.b.alpha32 + (size_t)c * D + dd) : 0.f;
  }
  if (x.nmma) {
    const int bi = acc_buf(rc, dbl);
    tacc = tmem + (uint32_t)(bi * 2 * tc.slot);
    mbar_wait(&tl.tfull[bi], rc.tf[bi] & 1);
    if (tr) tr[80] = clock64();
    fence_after_sync();
  }
  if (x.stage == 1) {
    const int n = x.rt * TM + r;
    float *Uh = p.b.Uh + (size_t)x.t * d.Pp * N, *Ul = p.b.Ul + (size_t)x.t * d.Pp * N;
    float *part = p.b.Upart + ((size_t)x.t * d.S1 + x.sp) * d.Pp * N;
    if (x.nmma) {
      for (int c0 = 0; c0 < ((p.dbg_flags & 64) ? 0 : x.nmma); c0 += 16) {
        float tot[16];
        acc_load16(tacc, ew, c0, nacc, tc.slot, tot);
        if (n < N) {
          // rows j0 + c0 + i of U (stride N); the columns past ncol (MMA padding) are not stored
          const int nv = min(16, x.ncol - c0);
          const uint32_t o0 = (uint32_t)(j0 + c0) * (uint32_t)N + (uint32_t)n;
          if (d.S1 == 1) {
            float *uh = Uh + o0, *ul = Ul + o0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (i < nv) {
                const float h = tf32_rna(tot[i]);
                uh[(uint32_t)i * (uint32_t)N] = h;
                ul[(uint32_t)i * (uint32_t)N] = tot[i] - h;
              }
            }
          } else {
            float *pp = part + o0;
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i < nv) pp[(uint32_t)i * (uint32_t)N] = tot[i];
          }
        }
      }
      fence_before_sync();
      __syncwarp();
      const int bi = acc_buf(rc, dbl);
      if (lane == 0) tempty_arrive<PR>(tl, bi, !dbl && tc.dbl);   // the MMA warp may overwrite the accumulator
      rc.tf[bi]++;
      rc.ti++;
      if (tr) tr[81] = clock64();
    }
    if (d.S1 > 1) {
      int rb, re;
      split_handoff(p, x, tl, &rb, &re);
      if (tr) tr[87] = clock64();
      if (x.mean && re > rb) {                 // Um: this CTA's share of the split partials
        const int n0 = x.rt * TM;
        const int nm = (re - rb) * d.Cp / 2;   // double2 elements of this share of Um
        const double *mbase = p.b.Umpart + (size_t)x.t * d.S1 * N * d.Cp;
        for (int e = et; e < nm; e += 128) {
          const size_t o = (size_t)(n0 + rb) * d.Cp + 2 * e;
          double2 v = make_double2(0.0, 0.0);
#pragma unroll 4
          for (int sidx = 0; sidx < d.S1; ++sidx) {
            const double2 pv = __ldcg(reinterpret_cast<const double2 *>(mbase + (size_t)sidx * N * d.Cp + o));
            v.x += pv.x;
            v.y += pv.y;
          }
          *reinterpret_cast<double2 *>(p.b.Um + (size_t)x.t * N * d.Cp + o) = v;
        }
      }
      if (x.nmma && re > rb) {
        const int n0 = x.rt * TM, r4n = (re - rb) >> 2;
        const size_t split = (size_t)d.Pp * N;
        const float *base = p.b.Upart + (size_t)x.t * d.S1 * split;
        const int tot4 = x.ncol * r4n;
        constexpr int V = 4;
        for (int e0 = et; e0 < tot4; e0 += 128 * V) {
          float4 acc4[V];
          size_t off[V];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int e = min(e0 + 128 * v, tot4 - 1);
            off[v] = (size_t)(j0 + e / r4n) * N + n0 + rb + 4 * (e % r4n);
            acc4[v] = __ldcg(reinterpret_cast<const float4 *>(base + off[v]));
          }
#pragma unroll 3
          for (int sidx = 1; sidx < d.S1; ++sidx) {
            float4 pv[V];
#pragma unroll
            for (int v = 0; v < V; ++v) pv[v] = __ldcg(reinterpret_cast<const float4 *>(base + sidx * split + off[v]));
#pragma unroll
            for (int v = 0; v < V; ++v) {
              acc4[v].x += pv[v].x; acc4[v].y += pv[v].y; acc4[v].z += pv[v].z; acc4[v].w += pv[v].w;
            }
          }
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (e0 + 128 * v < tot4) {
              float4 h;
              h.x = tf32_rna(acc4[v].x); h.y = tf32_rna(acc4[v].y); h.z = tf32_rna(acc4[v].z); h.w = tf32_rna(acc4[v].w);
              *reinterpret_cast<float4 *>(Uh + off[v]) = h;
              *reinterpret_cast<float4 *>(Ul + off[v]) =
                  make_float4(acc4[v].x - h.x, acc4[v].y - h.y, acc4[v].z - h.z, acc4[v].w - h.w);
            }
        }
      }
    }
    if (tr) tr[82] = clock64();
    return;
  }
  if (!x.nmma) return;
  // ---- stage 2: W = β acc + α_c ⊙ d for row dd, fp64 partial dᵀW per column (this tile) ----
  const int dd = x.rt * TM + r;
  const bool rv = dd < D;
  const float betaf = (float)p.beta;
  const size_t colbase = ((size_t)x.t * P + j0) * D + dd;
  const bool dts = tc.use_dtile;
  const float *dtile = reinterpret_cast<const float *>(sm + (size_t)rc.S * tc.stage_bytes);
  if (dts) {
    mbar_wait(&tl.dfull, rc.di & 1);
    rc.di++;
  }
  if (tr) tr[86] = clock64();
  // per 16-column group: W = β·acc + α_c ⊙ d, dot partials; the cluster of column j0 + c0 + i is
  // tracked incrementally (no integer division per column)
  const float *__restrict__ arow = p.b.alpha32 + dd;
  float *__restrict__ Wc = p.b.W + colbase;
  auto group_tot = [&](int c0, const float *dv, const float *tot) {
    // independent steps over the 16 columns (one epilogue warp per scheduler: ILP, not TLP, hides
    // latency): α, W, stores, exact fp64 products, then the butterfly reduction.  Columns of
    // retired probes get a W too (never read: the update skips them).
    float a[16], w[16];
    const int jc = j0 + c0, cl0 = jc / d.K;
    if (d.K >= 16) {
      // ≤ 2 clusters in a group of 16 columns: α of this row for both (read-only during the
      // E-step: the non-coherent path), column i of the group in cluster cl0 while i < nb
      const int nb = (cl0 + 1) * d.K - jc;
      const float a0 = rv ? __ldg(arow + (size_t)min(cl0, C - 1) * D) : 0.f;
      const float a1 = rv ? __ldg(arow + (size_t)min(cl0 + 1, C - 1) * D) : 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = i < nb ? a0 : a1;
    } else {
      int cl = cl0, rem = jc - cl0 * d.K;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        a[i] = rv ? __ldg(arow + (size_t)min(cl, C - 1) * D) : 0.f;
        if (++rem == d.K) { rem = 0; ++cl; }
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = fmaf(betaf, tot[i], a[i] * dv[i]);
    if (rv) {
      float *wc = Wc + (uint32_t)c0 * (uint32_t)D;
      const int nv = x.ncol - c0;            // the MMA padding columns past ncol are not stored
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nv) wc[(uint32_t)i * (uint32_t)D] = w[i];
    }
    double dot[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) dot[i] = (double)dv[i] * (double)w[i];
    int idx;
    const double sum = warp_reduce16(dot, lane, &idx);
    if ((lane & 1) == 0) tl.red[ew][c0 + idx] = sum;
  };
  auto group = [&](int c0, const float *dv) {
    float tot[16];
    acc_load16(tacc, ew, c0, nacc, tc.slot, tot);
    group_tot(c0, dv, tot);
  };
  if (p.dbg_flags & 64) {
    // diagnostic: accumulator not drained
  } else if (dts) {
    if (helped) {                             // the A warps take every other column group
      if (threadIdx.x == EPI0) tl.help_tacc = tacc;
      pair_sync();
      drain2_groups<CC>(p, tl, x, tacc, nacc, dtile, alpha, 0, 2);
      pair_sync();
    } else {
      drain2_groups<CC>(p, tl, x, tacc, nacc, dtile, alpha, 0, 1);
    }
  } else {
    // global loads of d: the next group's are issued while the current one is processed
    float dnx[16];
    auto load_d = [&](int c0, float *dst) {
      const uint32_t mk = c0 < x.nmma ? (mask[c0 >> 5] >> (c0 & 31)) & 0xFFFFu : 0u;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        dst[i] = (((mk >> i) & 1u) && rv) ? ldv(p.b.D32 + colbase + (size_t)(c0 + i) * D) : 0.f;
    };
    load_d(0, dnx);
    for (int c0 = 0; c0 < x.nmma; c0 += 16) {
      float dv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) dv[i] = dnx[i];
      load_d(c0 + 16, dnx);
      group(c0, dv);
    }
  }
  fence_before_sync();
  __syncwarp();
  {
    const int bi = acc_buf(rc, dbl);
    if (lane == 0) {
      tempty_arrive<PR>(tl, bi, !dbl && tc.dbl);
      if (dts) mbar_arrive(&tl.dempty);
    }
    rc.tf[bi]++;
    rc.ti++;
  }
  if (tr) tr[81] = clock64();
  epi_sync();
  for (int c = et; c < x.ncol && x.rt < d.nRT2; c += 128)
    if ((mask[c >> 5] >> (c & 31)) & 1u)
      stv(p.b.dAd + ((size_t)x.t * P + j0 + c) * d.nRT2 + x.rt,
          tl.red[0][c] + tl.red[1][c] + tl.red[2][c] + tl.red[3][c]);
  epi_sync();                                 // tl.red is reused by the next unit
  if (tr) tr[82] = clock64();
}

// ---------------------------------------------------------------------------------------------
// the persistent CG kernel: grid = #SMs (cooperative), 320 threads, one CTA per SM
// ---------------------------------------------------------------------------------------------
// PR: CTA pairs (2-CTA clusters, cta_group::2 MMAs of M = 256, each CTA staging half of B)
template <int CC, bool PR>
__global__ void __launch_bounds__(NTHREADS, 1) k_cg_persistent(KParams p, const __grid_constant__ TcMaps mp) {
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~(uintptr_t)1023);
  const Dims &d = p.d;
  const TcCfg &tc = p.tc;
  PSmemTail &tl = *reinterpret_cast<PSmemTail *>(sm + (size_t)tc.stages * tc.stage_bytes + tc.dtile_bytes);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, b = blockIdx.x;
  // units are dealt to GU dealers: the CTAs, or the CTA pairs (both CTAs of a pair walk the same units)
  const uint32_t rank = PR ? cluster_rank() : 0u;
  const int GU = PR ? G / 2 : G, bu = PR ? b / 2 : b;
  if (tid == 0) {
    for (int s = 0; s < tc.stages; ++s) {
      mbar_init(&tl.full[s], 1);
      mbar_init(&tl.bfull[s], 1);             // a pair's leader: its expect_tx; bytes of both CTAs' B halves
      mbar_init(&tl.empty[s], 5);             // the MMA warp's commit (or arrive) + the 4 A warps
      mbar_init(&tl.mdone[s], 4);             // the 4 epilogue warps' fp64 work on a mean chunk
    }
    for (int s = 0; s < tc.sa; ++s) {
      mbar_init(&tl.afull[s], PR ? 8 : 4);    // a pair's leader counts both CTAs' A warps
      mbar_init(&tl.aempty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tl.tfull[i], 1);
      mbar_init(&tl.tempty[i], PR ? 8 : 4);   // both CTAs' epilogue warps (leader's copy)
    }
    mbar_init(&tl.dfull, 1);
    mbar_init(&tl.dempty, 4);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&mp.phi); prefetch_tmap(&mp.phit); prefetch_tmap(&mp.u_hl); prefetch_tmap(&mp.d_hl);
    prefetch_tmap(&mp.dm); prefetch_tmap(&mp.um); prefetch_tmap(&mp.d32);
  }
  if (warp == 2) {
    if (PR) tmem_alloc_pair<512>(&tl.tslot);
    else tmem_alloc<512>(&tl.tslot);
  }
  fence_before_sync();
  __syncthreads();
  if (PR) cluster_sync_all();                 // the peer's barriers exist before any remote arrive
  fence_after_sync();
  const uint32_t tmem = tl.tslot;
  RingCtl rc{tc.stages, 0u, 0, 0u, tc.sa, 0u, 0, 0u, 0u, {0u, 0u}, {0u, 0u}, 0u, 0u, {0u, 0u, 0u, 0u, 0u, 0u}};
  unsigned epoch = 0;
  unsigned *bar = p.b.gridbar;
  const int nRTu1 = nrt_units(d.nRT1, PR), nRTu2 = nrt_units(d.nRT2, PR);
  const int n1 = d.Tl * d.nCT * nRTu1 * d.S1, n2 = d.Tl * d.nCT * nRTu2;
  // completion signals per task and stage (one per CTA and unit: a pair unit signals twice)
  const int E1 = d.nCT * nRTu1 * d.S1 * (PR ? 2 : 1), E2 = d.nCT * nRTu2 * (PR ? 2 : 1);
  int *cnt1 = p.b.dep, *cnt2 = p.b.dep + d.Tl;
  const int ncols = d.Tl * (d.P + d.C);
  const bool producer = warp == 0, issuer = warp == 1;
  const bool aw = warp >= 2 && warp < 6, epi = warp >= 6;
  const bool tile_role = true;
  // the A warps help drain a CTA's last stage-2 tile (the d tile path; not under diagnostics)
  const bool help2 = tc.use_dtile && !(p.dbg_flags & 64);
  for (int u = 0; u < d.cap; ++u) {
    if (b == 0 && tid == 0) p.b.ts[4 * u + 0] = globaltimer();
    // diagnostic trace of CTA 0's first unit of each phase at CG step trace_step (CMTCS_PHASE_LOG)
    unsigned long long *tr1 = (b == 0 && u == p.trace_step) ? p.b.ts + 4 * d.cap : nullptr;
    unsigned long long *tr2 = tr1 ? tr1 + 256 : nullptr;
    // ---- phase 1: U = Φ D ----
    if (tr1 && tid == 0) tr1[127] = clock64();   // trace times are SM clocks from here
    if (tile_role) {
      for (int w = bu; w < n1; w += GU, tr1 = nullptr) {
        Unit x = make_unit1(d, tc, w, GU, (int)rank);
        uint32_t mask[TC_NTMAX / 32];
        unit_work(p, x, lane, mask);
        if (!x.nmma && !x.mean) {
          if (tid == EPI0) dep_signal(cnt1 + x.t);
          continue;
        }
        if (producer) produce<PR>(p, mp, sm, tl, rc, x, tr1, rank);
        else if (issuer) mma_unit<PR>(p, sm, tl, rc, tmem, x, tr1, rank);
        else if (aw) a_unit<PR>(p, sm, tl, rc, tmem, x, (tr1 && threadIdx.x == AW0) ? tr1 : nullptr, nullptr);
        else if (epi) {
          probe_epilogue<CC, PR>(p, sm, tl, rc, tmem, x, mask, tr1, false);
          epi_sync();                         // this tile's U / Um stores, then EPI0's release
          if (tid == EPI0) dep_signal(cnt1 + x.t);
        }
      }
    }
    // no grid barrier: a stage-2 unit of task t starts once task t's stage-1 units are complete
    if (tid == EPI0) atomicMax(p.b.ts + 4 * u + 3, globaltimer());
    // ---- phase 2: W = βΦᵀU + αD, dᵀW partials ----
    if (tr2 && tid == 0) tr2[127] = clock64();
    if (tile_role) {
      for (int w = bu; w < n2; w += GU, tr2 = nullptr) {
        Unit x = make_unit2(d, tc, w, GU, (int)rank);
        uint32_t mask[TC_NTMAX / 32];
        unit_work(p, x, lane, mask);
        if (!x.nmma && !x.mean) {
          if (tid == EPI0) dep_signal(cnt2 + x.t);
          continue;
        }
        if (producer) {
          if (lane == 0) dep_wait(cnt1 + x.t, (u + 1) * E1);   // U, Um of task t complete
          __syncwarp();
          fence_proxy_async_global();         // the acquired generic writes → this warp's TMA reads
          produce<PR>(p, mp, sm, tl, rc, x, tr2, rank);
        }
        else if (issuer) mma_unit<PR>(p, sm, tl, rc, tmem, x, tr2, rank);
        else if (aw) {
          a_unit<PR>(p, sm, tl, rc, tmem, x, (tr2 && threadIdx.x == AW0) ? tr2 : nullptr, tr2 ? tr2 + 160 : nullptr);
          if (help2 && x.nmma && (w + GU >= n2 || help_mean(p, x))) a_help_drain2<CC>(p, sm, tl, rc, x);
        }
        else if (epi) {
          if (tid == EPI0 && x.rt == 0 && x.nmma) atomicAdd(p.b.histp + u, x.nmma);
          probe_epilogue<CC, PR>(p, sm, tl, rc, tmem, x, mask, tr2, help2 && (w + GU >= n2 || (x.nmma && help_mean(p, x))));
          epi_sync();                         // this tile's W / Wm / dᵀAd stores, then EPI0's release
          if (tid == EPI0) dep_signal(cnt2 + x.t);
        }
      }
    }
    // no grid barrier: the update of a column of task t starts once task t's stage-2 units are done
    if (tid == EPI0) atomicMax(p.b.ts + 4 * u + 1, globaltimer());
    __syncthreads();                          // the ring's shared memory is reused by the update
    // ---- phase 3: CG update, one warp per active column ----
    unsigned long long *tr3 = (b == 0 && u == p.trace_step && warp == 0) ? p.b.ts + 4 * d.cap + 160 : nullptr;
    if (tr3 && lane == 0) tr3[8] = clock64();
    float4 *stage_d = (size_t)NTHREADS / 32 * 2 * d.D * 4 <= (size_t)tc.stages * tc.stage_bytes
                          ? reinterpret_cast<float4 *>(sm) + (size_t)warp * (d.D / 2) : nullptr;
    for (int w = b * (NTHREADS / 32) + warp; w < ncols; w += G * (NTHREADS / 32)) {
      const int t = w / (d.P + d.C), j = w % (d.P + d.C);
      // the column's flag is written only by this warp's own update (the same column every step):
      // read it before the wait, and issue the task-activity mark early (its result is used last)
      const bool active = j < d.P ? ldv(p.b.flag + (size_t)t * d.P + j) == 1
                                  : ldv(p.b.flagm + (size_t)t * d.C + (j - d.P)) == 1;
      const int tm_old = (active && lane == 0) ? atomicMax(p.b.tmark + t, u + 1) : u + 1;
      if (lane == 0) dep_wait(cnt2 + t, (u + 1) * E2);   // W, dᵀAd of task t complete
      __syncwarp();
      if (j < d.P) {
        if (active) {
          if (lane == 0) atomicAdd(p.b.hist + u, 1);
          update_probe(p, t, j, u, lane, stage_d, (tr3 && w == b * (NTHREADS / 32) + warp && lane == 0) ? tr3 : nullptr);
        }
      } else {
        if (active) {
          if (lane == 0) atomicAdd(p.b.histm + u, 1);
          update_mean(p, t, j - d.P, u, lane);
        }
      }
      if (tm_old < u + 1) atomicAdd(p.b.histt + u, 1);
    }
    grid_sync(bar, epoch);
    if (b == 0 && tid == 0) {
      p.b.ts[4 * u + 2] = globaltimer();
      *p.b.u = u + 1;                          // CG steps executed
    }
    if (ldv(p.b.alive + u) == 0) break;     // grid-uniform: every CTA reads the settled count
  }
  fence_before_sync();
  __syncthreads();
  if (PR) {
    cluster_sync_all();                       // the peer is done with this pair's tensor memory
    if (warp == 2) tmem_dealloc_pair<512>(tmem);
  } else if (warp == 2) {
    tmem_dealloc<512>(tmem);
  }
}

// Φᵀ (fp32) of every task, once at init: the K-major A operand of stage 2.  32×32 smem-tiled transpose.
__global__ void k_transpose_phi(const float *__restrict__ phi, int rows, int cols, float *__restrict__ phit) {
  __shared__ float tile[32][33];
  const int mat = blockIdx.z;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const float *src = phi + (size_t)mat * rows * cols;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? src[(size_t)r * cols + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;   // transposed: row c, column r
    if (c < cols && r < rows) phit[(size_t)mat * rows * cols + (size_t)c * rows + r] = tile[threadIdx.x][i];
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 3-D tensor map over [mats][rows][cols] row-major (one matrix per task); box box_cols × box_rows × 1
bool encode_3d(EncodeTiledFn enc, CUtensorMap *m, const void *ptr, CUtensorMapDataType dt, int esize, long mats,
               long rows, long cols, int box_cols, int box_rows, bool swizzle) {
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)mats};
  cuuint64_t strides[2] = {(cuuint64_t)cols * esize, (cuuint64_t)rows * cols * esize};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, dt, 3, const_cast<void *>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D view [2][mats][rows][cols] of two equally shaped fp32 arrays (hi at `hi`, lo at `lo`, lo − hi a
// multiple of 16 bytes), box box_cols × box_rows × 1 × 2, 128-byte swizzle: one TMA brings a task's
// hi tile and then its lo tile
bool encode_hilo(EncodeTiledFn enc, CUtensorMap *m, const float *hi, const float *lo, long mats, long rows,
                 long cols, int box_cols, int box_rows) {
  const long long gap = (long long)((const char *)lo - (const char *)hi);
  if (gap <= 0 || gap % 16) return false;
  cuuint64_t dims[4] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)mats, 2};
  cuuint64_t strides[3] = {(cuuint64_t)cols * 4, (cuuint64_t)rows * cols * 4, (cuuint64_t)gap};
  cuuint32_t box[4] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1, 2};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(hi), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

size_t tc_smem_bytes(const TcCfg &tc, int P) {
  (void)P;
  return 1024 + (size_t)tc.stages * tc.stage_bytes + tc.dtile_bytes + sizeof(PSmemTail);
}

bool encode_maps(const KParams &p, TcMaps *m, char *why) {
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
      q != cudaDriverEntryPointSuccess) {
    snprintf(why, 256, "cuTensorMapEncodeTiled unavailable");
    return false;
  }
  EncodeTiledFn enc = (EncodeTiledFn)fn;
  const Dims &d = p.d;
  const Bufs &b = p.b;
  const long mats = d.shared_phi ? 1 : d.Tl;
  const CUtensorMapDataType F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32, F64 = CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  const int NT = p.tc.NT;
  const long Tl = d.Tl;
  const bool ok = encode_3d(enc, &m->phi, p.phi, F32, 4, mats, d.N, d.D, 32, TM, true) &&
                  encode_3d(enc, &m->phit, b.PT, F32, 4, mats, d.D, d.N, 32, TM, true) &&
                  encode_3d(enc, &m->dm, b.Dm, F64, 8, Tl, d.C, d.D, TK, d.C, false) &&
                  encode_3d(enc, &m->um, b.Um, F64, 8, Tl, d.N, d.Cp, d.Cp, TK, false) &&
                  encode_3d(enc, &m->d32, b.D32, F32, 4, Tl, d.P, d.D, TM, NT, false) &&
                  encode_hilo(enc, &m->u_hl, b.Uh, b.Ul, Tl, d.Pp, d.N, 32, p.tc.pair ? NT / 2 : NT) &&
                  encode_hilo(enc, &m->d_hl, b.Dh, b.Dl, Tl, d.P, d.D, 32, p.tc.pair ? NT / 2 : NT);
  if (!ok) snprintf(why, 256, "cuTensorMapEncodeTiled failed");
  return ok;
}

// kernel instantiation for the cluster count: CC ∈ {4, 8, 16} bounds C at compile time
typedef void (*CgKernel)(KParams, const TcMaps);
CgKernel cg_kernel(int C, int pair) {
  if (pair) {
    if (C <= 4) return k_cg_persistent<4, true>;
    if (C <= 8) return k_cg_persistent<8, true>;
    return k_cg_persistent<16, true>;
  }
  if (C <= 4) return k_cg_persistent<4, false>;
  if (C <= 8) return k_cg_persistent<8, false>;
  return k_cg_persistent<16, false>;
}

int cg_grid_size(const KParams &p) {
  int dev = 0, sms = 0, occ = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  const size_t smem = tc_smem_bytes(p.tc, p.d.P);
  const CgKernel k = cg_kernel(p.d.C, p.tc.pair);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NTHREADS, smem) != cudaSuccess) return 0;
  if (occ < 1) return 0;
  if (!p.tc.pair) return sms;  // one CTA per SM (512 TMEM columns each)
  // CTA pairs: as many 2-CTA clusters as can be co-resident (every CTA must be resident: grid barrier)
  if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 0) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms / 2 * 2);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, k, &cfg) != cudaSuccess) return 0;
  return std::min(sms / 2, clusters) * 2;
}

cudaError_t launch_split_phi(const KParams &p, cudaStream_t s) {
  const int mats = p.d.shared_phi ? 1 : p.d.Tl;
  dim3 grid((p.d.D + 31) / 32, (p.d.N + 31) / 32, mats);
  k_transpose_phi<<<grid, dim3(32, 8), 0, s>>>(p.phi, p.d.N, p.d.D, p.b.PT);
  return cudaGetLastError();
}

cudaError_t launch_cg_persistent(const KParams &p, const TcMaps &maps, int grid, cudaStream_t s) {
  const size_t smem = tc_smem_bytes(p.tc, p.d.P);
  cudaError_t e = cudaMemsetAsync(p.b.gridbar, 0, sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(p.b.dep, 0, sizeof(int) * 2 * p.d.Tl, s);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;   // co-residency of all CTAs (grid barriers)
  attr[0].val.cooperative = 1;
  int na = 1;
  if (p.tc.pair) {   // 2-CTA clusters (the grid is sized to the co-resident cluster count)
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, cg_kernel(p.d.C, p.tc.pair), p, maps);
}

}  // namespace cmtcs
