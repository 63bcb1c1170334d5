// Internal declarations shared by the libcmtcs translation units (not part of the C ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "cmtcs.h"

namespace cmtcs {

constexpr int MAXC = 16;        // clusters supported by the fp64 mean-column tiles
constexpr int OP_BR = 128;      // operator tile rows (N in stage 1, D in stage 2)
constexpr int OP_BK = 16;       // mean-column (SIMT) contraction chunk
constexpr int OP_THREADS = 256; // mean-column kernels
constexpr int TC_THREADS = 128; // tensor-core probe kernels (4 warps = 128 TMEM lanes)
constexpr int TC_NTMAX = 128;   // widest probe-column tile (MMA N; TMEM also holds the A stages)

// Sizes of one rank's problem.  Column index of probe (c, k) inside a task: col = c*K + k.
struct Dims {
  int T, Tl, t0, N, D, C, K;
  int P;     // probe columns per task = C*K
  int Pp;    // P rounded up to a multiple of 4 (row stride of U)
  int ldv;   // FP32 engine: row stride of its d-major probe vectors X, R, D32, W [D][T_loc·Pp] and of U
             // [N][T_loc·Pp] (column g = t·Pp + j); 0 for the column-contiguous layouts [T_loc][P][D]
  int Cp;    // C rounded up to even (row stride of Um: 16-byte TMA rows)
  int cap;   // CG step cap U
  int nw;    // 64-bit probe words per column = ceil(D/64)
  int nRT1;  // stage-1 row tiles  = ceil(N / OP_BR)
  int nRT2;  // stage-2 row tiles  = ceil(D / OP_BR)
  int nCT;   // probe column tiles = ceil(P / TcCfg::NT)
  int S1;    // stage-1 split-K factor (balances the persistent grid when T·N is small)
  int K1;    // stage-1 contraction length per split (multiple of OP_BK)
  int split_coop;  // S1 > 1 with every stage-1 unit co-resident: split CTAs reduce cooperatively
  int pair;        // CTA-pair operator (TcCfg::pair), decided with the split: pairs need S1 = 1
  int shared_phi;
  int64_t phi_task_stride;  // elements between Φ_t and Φ_{t+1} (0 if shared)
  int op;          // CMTCS_OP_DENSE (Φ_t a matrix, tensor cores), CMTCS_OP_DENSE_FP32 (the same on the FP32
                   // CUDA cores, k_simt.cu) or CMTCS_OP_PARTIAL_FOURIER (Φ_t = Ω_t F, k_fourier.cu)
};

// Device buffers carved from the caller's workspace (all sizes in DESIGN.md §5).
struct Bufs {
  double *alpha64;   // [C][D]
  float *alpha32;    // [C][D]
  double *logsum_alpha;  // [C]  Σ_d log α_cd
  double *logpi;     // [C]
  double *b64;       // [Tl][D]   βΦᵀy
  double *bnorm2;    // [Tl]      ‖b‖²
  float *X, *R, *W;  // probe columns [Tl][P][D]; W = Ad
  float *D32;        // probe directions d [Tl][P][D] (fp32: the epilogue's d tile, the update)
  float *Dh, *Dl;    // the same as the exact tf32 pair d = Dh + Dl (stage-1 B operand) [Tl][P][D]
  float *PT;         // Φᵀ fp32 [Tl or 1][D][N] (stage-2 A operand; stage 1 reads the caller's Φ)
  double *Xm, *Rm, *Dm, *Wm; // mean columns  [Tl][C][D]
  float *Uh, *Ul;    // stage-1 output U = ΦD as the exact tf32 pair (stage-2 B operand), [Tl][Pp][N]
  double *Um;        // [Tl][N][Cp]
  double *rr;        // [Tl][P]
  double *rrm;       // [Tl][C]
  double *dAd;       // [Tl][P][nRT2]  per-row-tile partial dᵀAd
  double *dAdm;      // [Tl][C][nRT2]
  int *flag;         // [Tl][P]  1 = active
  int *flagm;        // [Tl][C]
  int *steps;        // [Tl][P]
  int *stepsm;       // [Tl][C]
  int *act;          // [Tl][P]  compacted active probe columns (ascending)
  int *m_act;        // [Tl]
  double *gam, *xi;  // [Tl*P][cap]
  double *tau;       // [Tl*P]
  double *s;         // [Tl][C][D]
  double *nu, *ell, *q;  // [Tl][C]
  double *ll;        // [Tl]
  double *red;       // [C*D + C + 1]  Eq. 4 sums (den, num) and Σ_t log p(y_t)
  double *red_local; // [C*D + C + 1]  the same before the all-reduce (this rank's tasks)
  int *alive;        // [2·cap]  columns still active after step u (FP32 engine: one [cap] array per task half)
  int *hist;         // [cap]  probe columns active at step u
  int *histm;        // [cap]  mean columns active at step u
  int *histt;        // [cap]  tasks with an active column at step u
  int *histp;        // [cap]  probe columns the operator multiplied at step u (MMA widths of the
                     //        column tiles with ≥ 1 active column, per task: padded work)
  int *status;       // [8]    first error: code, t, col, u
  int *u;            // [1]    current CG step (device-side loop counter of the CG graph)
  unsigned long long *ts;  // [cap][4] per-step %globaltimer stamps taken by CTA 0 after the grid
                           //          barriers: step start, operator done, update done, unused
  double *stats;     // [16]   step statistics (filled by k_stats)
  float *Upart;      // [Tl][S1][Pp][N]  stage-1 split-K partial tiles (S1 > 1)
  double *Umpart;    // [Tl][S1][N][Cp]
  int *tmark;        // [Tl]   last CG step (+1) at which the task had an active column
  int *tilecnt;      // [Tl][nCT][nRT1]  split-K arrival counters (self re-arming)
  unsigned *gridbar; // [1]    grid-barrier arrival counter of the persistent CG kernel
  int *dep;          // [2][Tl] per-task completion counters of stage 1 / stage 2 units (monotonic)
  int *assign;       // [Tl]
  double *resm;      // [Tl][C]  ‖y_t − Φ_t μ_tc‖² (partial-Fourier path; the dense path uses Um)
  double *ftw;       // [2·D]    partial Fourier: per-stage twiddles tw2[h + pos] = exp(−2πi pos/2h), fp64 pairs
};

// tensor-core operator configuration (chosen at init from P)
struct TcCfg {
  int NT;            // column tile width (multiple of 16, ≤ TC_NTMAX)
  int slot;          // TMEM columns per accumulator (NT rounded up to 16)
  int sa;            // A stages in TMEM (64 columns each: the tf32 hi and lo halves of a 128 × 32 tile)
  int acol0;         // first TMEM column of the A stages (= 512 − 64·sa; accumulators below)
  int dbl;           // two accumulator buffers (cross + one main each) fit below acol0
  int nacc;          // K-split main accumulators ((1 + nacc)·slot ≤ acol0)
  int stages;        // smem pipeline depth
  unsigned stage_bytes;
  int pf;            // L2 prefetch distance of the A tiles (chunks ahead of the one being loaded; 0 = off)
  int l2hint;        // TMA L2 cache hints: A tiles evict-first, B tiles evict-last (CMTCS_L2HINT)
  int pair;          // CTA pairs: 2-CTA clusters issuing cta_group::2 MMAs (M = 256 rows: a row-tile
                     // pair), each CTA staging half of the tile's B columns
  int use_dtile;     // stage-2 epilogue reads its d tile (NT × 128 fp32) from smem, staged by TMA
  unsigned dtile_bytes;
};

// TMA descriptors (host-encoded, passed as a __grid_constant__ kernel parameter)
struct TcMaps {
  // every map is per task, [task][rows][cols] (box depth 1 in the task dimension): a tile or K chunk
  // overhanging a task's matrix is zero-filled instead of reading the next task's data
  CUtensorMap phi;             // fp32 Φ (the caller's) [Tl or 1][N][D], box 32 × 128, SW128
  CUtensorMap phit;            // fp32 Φᵀ [Tl or 1][D][N], box 32 × 128, SW128
  CUtensorMap dm;              // fp64 [Tl][C][D], box 32 × C (mean directions)
  CUtensorMap um;              // fp64 [Tl][N][Cp], box Cp × 32 (Φ·d of the mean columns)
  CUtensorMap d32;             // fp32 [Tl][P][D], box 128 × NT (probe directions, epilogue)
  CUtensorMap u_hl, d_hl;      // U = ΦD [Tl][Pp][N] and the directions [Tl][P][D] as their exact tf32
                               // pairs, hi and lo arrays viewed as one 4-D tensor [2][Tl][rows][cols],
                               // box 32 × NT × 1 × 2: both B tiles of a stage with one TMA
};

struct KParams {
  Dims d;
  Bufs b;
  TcCfg tc;
  const float *phi;
  const float *y;
  const int *rows;             // partial Fourier: sampled DFT rows [Tl][N] (Ω_t)
  double beta;
  double tol;                  // probe columns: stop when ‖r‖ ≤ tol·‖p‖
  double tol_mean;             // mean columns
  double alpha_max, var_floor, empty_eps;
  uint64_t seed;
  int it;                      // global EM iteration index of this E-step
  const uint64_t *probe_bits;  // optional override
  const double *q_override;    // optional
  int toff, tcnt;              // FP32 engine: the task window [toff, toff + tcnt) of this launch (tcnt = 0: all tasks)
  int learn_pi;                // M-step also sets log π_c = log((1/T) Σ_t q_tc) (reading P1)
  int trace_step;              // CMTCS_TRACE_STEP (default 5): the CG step CMTCS_PHASE_LOG traces
  int dbg_flags;               // CMTCS_DBG (diagnostics only, wrong results): 1 no DMMA, 2 no tcgen05.mma,
                               // 4 no tf32 split, 8/16/32 accumulator layouts, 64 no epilogue, 128 no TMA;
                               // (results unchanged:) 4096 no 2-MMA form, 16384 no A-warp drain help on mean units;
                               // 65536 probe columns never break down (timing runs with the flags above)
};

// launchers (return cudaGetLastError())
cudaError_t launch_init_columns(const KParams &p, cudaStream_t s);
cudaError_t launch_split_phi(const KParams &p, cudaStream_t s);
size_t tc_smem_bytes(const TcCfg &tc, int P);
int cg_grid_size(const KParams &p);   // CTAs of the persistent CG kernel (one per SM), 0 on failure
cudaError_t launch_cg_persistent(const KParams &p, const TcMaps &maps, int grid, cudaStream_t s);
bool encode_maps(const KParams &p, TcMaps *maps, char *why);   // after the workspace is carved
cudaError_t launch_mu_stage1(const KParams &p, const double *mu_src, cudaStream_t s);
cudaError_t launch_rhs(const KParams &p, cudaStream_t s);
cudaError_t launch_alpha_stats(const KParams &p, cudaStream_t s);
cudaError_t launch_diag(const KParams &p, cudaStream_t s);
cudaError_t launch_lanczos(const double *gam, const double *xi, const int *steps, int n, int ld,
                           int D, double *tau, double *scratch, int *status, cudaStream_t s);
cudaError_t launch_estep_finish(const KParams &p, cudaStream_t s);
cudaError_t launch_mstep_partial(const KParams &p, cudaStream_t s);
cudaError_t launch_mstep_finish(const KParams &p, cudaStream_t s);
cudaError_t launch_stats(const KParams &p, cudaStream_t s);
cudaError_t launch_readout(const KParams &p, double *recon, cudaStream_t s);
cudaError_t launch_probe_words(uint64_t seed, int it, int T, int t0, int Tl, int C, int K, int D,
                               uint64_t *out, cudaStream_t s);
cudaError_t launch_copy_transcript(const KParams &p, double *gam, double *xi, cudaStream_t s);
bool fourier_supported(int D, int N, char *why);
cudaError_t launch_fourier_rhs(const KParams &p, cudaStream_t s);
cudaError_t launch_fourier_cg(const KParams &p, int sms, cudaStream_t s);
// CG loop of an E-step with the operator on the FP32 CUDA cores (op_kind = CMTCS_OP_DENSE_FP32, k_simt.cu)
struct SimtTiming {                 // live timing of the FP32 engine (cmtcs_set_timing): CUDA events per step
  static constexpr int B = 8;       // steps between host termination checks (event pool of B steps)
  cudaEvent_t ev[3 * B];            // operator start, update start, update end
  double op_ms, upd_ms;
};
struct SimtStreams {                // the FP32 engine's side stream: the fp64 mean-column kernels run
  cudaStream_t side;                // beside the probe SGEMMs (fork after the update, join before it);
  cudaEvent_t fork, join;           // with two task halves (run_simt_cg) it carries the second half's CG loop
};
cudaError_t run_simt_cg(const KParams &p, int *h_alive, int64_t *launches, SimtTiming *tm, const SimtStreams &ss,
                        cudaStream_t s);

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// error codes written to status[0] by kernels
enum { ST_OK = 0, ST_BREAKDOWN = 1, ST_EIG = 2, ST_NUMERIC = 3 };

}  // namespace cmtcs
