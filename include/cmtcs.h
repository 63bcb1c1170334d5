/*
 * cmtcs.h — C ABI of the B200-native CoFEM hot path (covariance-free EM for clustered
 * multi-task compressive sensing, arXiv 2310.00420).  libcmtcs.so implements it with
 * hand-written sm_100a kernels; NCCL performs the one collective per EM iteration.
 *
 * Operation (PAPER.md citations are lines of the paper's LaTeX source):
 *   model           PAPER.md:24-30 (Eq. 1): y_t = Φ_t z_t + ε, z_t | a_t=c ~ N(0, diag(α_c)^-1)
 *   E-step          PAPER.md:45-59 (Eq. 3) and Alg. 2 lines 3-13:
 *                   per task t and cluster c, batched CG (Alg. 1) on
 *                   A_tc = βΦ_tᵀΦ_t + diag(α_c) with 1 mean RHS βΦ_tᵀy_t and K Rademacher
 *                   probes (Eq. 6); s_tc (Eq. 5); ν̄_tc ≈ log det Σ_tc
 *                   by Lanczos quadrature on the CG transcript (Eq. 7-9);
 *                   q_t = softmax_c(½ℓ_tc + log π_c) (Eq. 3).
 *   M-step          PAPER.md:63 (Eq. 4): α_cd = Σ_t q_tc / Σ_t q_tc (μ_tcd² + s_tcd),
 *                   sums all-reduced over ranks (one ncclAllReduce per EM iteration).
 *   readout         Alg. 2 lines 17-20: a_t = argmax_c q_tc, ẑ_t = μ_{t,a_t}.
 * No D×D matrix is ever formed.  Readings of silent/ambiguous points: DESIGN.md §3.
 *
 * Conventions.  Every function returns cmtcs_status (0 = OK); none throws, aborts or exits.
 * "device" pointers are CUDA global-memory pointers on the context's device; "host" pointers
 * are ordinary CPU memory.  All work is enqueued on the caller's CUDA stream; em_step
 * synchronises that stream once per call (to return `info`).  After any error other than
 * EINVAL from argument checking, the context is in CMTCS_ESTATE until destroyed, and
 * cmtcs_last_error() describes the failure (with (task, column, step) for breakdowns).
 * Precision: probe columns are fp32 vectors with fp64 scalars (γ, ξ, dot products); the mean
 * columns, log-det quadrature, responsibilities and M-step are fp64.
 */
#ifndef CMTCS_H
#define CMTCS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CMTCS_OK = 0,
  CMTCS_EINVAL = 1,     /* bad argument / dimension / α ≤ 0 / π not a distribution          */
  CMTCS_ENOMEM = 2,     /* workspace too small                                              */
  CMTCS_ECUDA = 3,      /* CUDA runtime error                                               */
  CMTCS_ENCCL = 4,      /* NCCL error                                                       */
  CMTCS_EBREAKDOWN = 5, /* CG breakdown dᵀAd ≤ 0 (Alg. 1 line 3)                */
  CMTCS_EEIG = 6,       /* tridiagonal eigen-iteration failed or Ritz value ≤ 0 (Eq. 8-9)   */
  CMTCS_ENUMERIC = 7,   /* NaN/Inf in ℓ, or softmax over all −∞ (Eq. 3)                     */
  CMTCS_ESTATE = 8      /* context unusable after an earlier error                          */
} cmtcs_status;

/* Problem statement (PAPER.md:12-13, 24-30 for Φ_t, y_t, β, π, C; PAPER.md:72, 80 for K, U). */
typedef struct cmtcs_problem {
  int32_t T;             /* global number of tasks (probe streams are indexed by global t)     */
  int32_t N, D;          /* measurements and signal dimension; N % 4 == 0 and D % 4 == 0        */
  int32_t C;             /* clusters, 1 ≤ C ≤ 16                                                */
  int32_t K;             /* Rademacher probes per (t, c), K ≥ 1                                 */
  int32_t shared_phi;    /* 1: one Φ [N][D] shared by all tasks; 0: Φ_t per task               */
  double beta;           /* noise precision β = 1/σ² > 0                                        */
  const double *pi;      /* host, C entries > 0 summing to 1 ± 1e-9: the prior π,
                            fixed, or the initial value when learn_pi = 1                         */
  int32_t cg_max_iters;  /* U: CG step cap per system, ≥ 1                                      */
  double cg_rel_tol;     /* ≥ 0: a column stops after step u when ‖r_{u+1}‖₂ ≤ tol·‖b‖₂         */
  double alpha_max;      /* α cap (1e12)                                                        */
  double var_floor;      /* s clamp inside Eq. 4 only (1e-12)                                   */
  double empty_eps;      /* Σ_t q_tc below this keeps α_c (1e-10)                               */
  uint64_t probe_seed;   /* root of the counter-based probe hash (reading A6)         */
  int32_t task_begin;    /* this rank owns global tasks [task_begin, task_end)                  */
  int32_t task_end;
  int32_t em_iter0;      /* global EM-iteration index of the next em_step (probe counter `it`) */
  double mean_rel_tol;   /* tolerance of the C mean systems A μ = βΦᵀy; < 0 ⇒ cg_rel_tol.  A tighter
                            value (e.g. 1e-10) makes μ independent of where CG stops (DESIGN.md §3 A5) */
  int32_t op_kind;       /* CMTCS_OP_DENSE: Φ_t is the caller's matrix (phi).  CMTCS_OP_PARTIAL_FOURIER:
                            the paper's §4 sensing matrix Φ_t = Ω_t F — F the unitary
                            D-point DFT, Ω_t the N rows fourier_rows[t] of the identity, real-embedded as
                            [Re(Ω_t F); Im(Ω_t F)] (reading F1), applied by FFT; then phi must
                            be NULL, y is [T_loc][2N] (N real parts, then N imaginary parts), D is a
                            power of two in [512, 8192] and shared_phi = 0                           */
  const int32_t *fourier_rows; /* device, BORROWED, op_kind = PARTIAL_FOURIER: int32 [T_loc][N], distinct
                            rows in [0, D) per task (must outlive ctx); NULL otherwise                */
  int32_t learn_pi;      /* 0: π fixed (the paper's setting).  1: π is learned — every
                            M-step also sets π_c = (1/T) Σ_t q_tc over all T tasks (all ranks: the
                            Σ_t q_tc of the Eq. 4 all-reduce), the mixture-weight M-step PAPER.md:30
                            points to ("can also be learned", McLachlan); the next E-step's Eq. 3
                            softmax uses it (reading P1).  An emptied cluster gets π_c = 0
                            (log π_c = −∞, q_tc = 0 from then on).                                  */
} cmtcs_problem;

/* CMTCS_OP_DENSE_FP32: the same dense Φ_t as CMTCS_OP_DENSE, the operator on the FP32 CUDA cores
 * (round-to-nearest FFMA accumulation) instead of the 3xTF32 tensor cores.  The north_star allows
 * the tensor path "only if the oracle tolerance holds": tcgen05's truncating fp32 accumulation
 * biases ν̄ and misses |ΔL| ≤ 1e-3 at configs 4-5; this operator meets it. */
enum { CMTCS_OP_DENSE = 0, CMTCS_OP_PARTIAL_FOURIER = 1, CMTCS_OP_DENSE_FP32 = 2 };

/* Statistics of the last EM iteration run by cmtcs_em_step (host struct, filled on return). */
typedef struct cmtcs_step_info {
  double loglik;             /* L(θ̂) = (1/T)Σ_t log p(y_t|θ̂) at the entry α, all ranks */
  int32_t em_iter;           /* global index of that EM iteration                              */
  int32_t cg_iters;          /* CG iterations executed (max steps over this rank's columns)    */
  int32_t mu_steps_min, mu_steps_max;
  int32_t probe_steps_min, probe_steps_max;
  double probe_steps_mean;
  int64_t n_cap_hit;         /* columns (mean + probe) that stopped at the cap unconverged     */
  int64_t probe_col_iters;   /* Σ_u (#active probe columns at step u), this rank               */
  int64_t mean_col_iters;    /* Σ_u (#active mean columns at step u), this rank                */
  int64_t task_iters;        /* Σ_u (#tasks with ≥ 1 active column at step u), this rank       */
  int64_t kernel_launches;   /* kernels this library launched during the call                  */
  int64_t tile_col_iters;    /* Σ_u probe columns the operator multiplied at step u: the MMA
                                widths of every column tile with ≥ 1 active column (retired
                                columns inside such a tile are multiplied too; padded work ≥
                                probe_col_iters), this rank                                      */
} cmtcs_step_info;

typedef struct cmtcs_ctx cmtcs_ctx;

/* NCCL unique id (128 bytes) for a multi-rank context; call on rank 0 and broadcast. */
cmtcs_status cmtcs_get_unique_id(uint8_t out[128]);

/* Bytes of device workspace cmtcs_init needs for problem p (shard of p->task_begin..end). */
cmtcs_status cmtcs_workspace_size(const cmtcs_problem *p, size_t *bytes);

/* Create a context.
 *   phi      device, BORROWED (must outlive ctx): fp32 [T_loc][N][D] row-major, or [N][D] if
 *            p->shared_phi; T_loc = task_end − task_begin, task i is global task task_begin+i.
 *            NULL for op_kind = CMTCS_OP_PARTIAL_FOURIER (Φ_t from p->fourier_rows).
 *   y        device, BORROWED: fp32 [T_loc][N] ([T_loc][2N] for the partial-Fourier operator).
 *   alpha0   host or device, COPIED: fp64 [C][D], every entry > 0 (α₀, Alg. 2 line 1).
 *   workspace device, BORROWED, ≥ cmtcs_workspace_size bytes, 256-byte aligned.
 *   nccl_uid NULL with world == 1 for a single GPU; else the rank-0 id, rank in [0, world).  A uid
 *            with world == 1 creates a 1-rank communicator, so the Eq. 4 all-reduce runs through
 *            NCCL on one GPU (tests of the NCCL path where only one GPU exists).
 *   device   CUDA device ordinal; cuda_stream a cudaStream_t (NULL = legacy default stream).
 * Computes b_t = βΦ_tᵀy_t (Eq. 6) once.  EINVAL on any bad argument (nothing allocated). */
cmtcs_status cmtcs_init(cmtcs_ctx **ctx, const cmtcs_problem *p, const float *phi,
                        const float *y, const double *alpha0, void *workspace,
                        size_t workspace_bytes, const uint8_t *nccl_uid, int32_t rank,
                        int32_t world, int32_t device, void *cuda_stream);

/* Run n_iters EM iterations (Alg. 2 lines 2-16): E-step at the current α, all-reduce of the
 * Eq. 4 sums, α update.  probe_bits (device, optional, requires n_iters == 1) overrides the
 * hash: uint64 [T_loc][C][K][ceil(D/64)], bit (d mod 64) of word ⌊d/64⌋ set ⇔ p_d = −1.
 * q_override (device, optional, requires n_iters == 1): fp64 [T_loc][C] used by the M-step in
 * place of the computed q (the computed q is still reported).  info (host, may be NULL). */
cmtcs_status cmtcs_em_step(cmtcs_ctx *ctx, int32_t n_iters, const uint64_t *probe_bits,
                           const double *q_override, cmtcs_step_info *info);

/* Copy the last E-step's posterior and the current α into caller buffers (device; NULL skips):
 *   mu fp64 [T_loc][C][D], s fp64 [T_loc][C][D] (Eq. 5, unclamped), logdet fp64 [T_loc][C] (ν̄),
 *   q fp64 [T_loc][C], alpha fp64 [C][D] (after the last M-step), assign int32 [T_loc]
 *   (argmax, ties → lowest c), recon fp64 [T_loc][D] = μ_{t,a_t}.  ESTATE before any em_step. */
cmtcs_status cmtcs_posterior(cmtcs_ctx *ctx, double *mu, double *s, double *logdet, double *q,
                             double *alpha, int32_t *assign, double *recon);

/* The current mixture weights π (fp64 [C], host or device): the initial p->pi, or after each
 * M-step with learn_pi the learned ones.  ESTATE on an unusable context. */
cmtcs_status cmtcs_get_pi(cmtcs_ctx *ctx, double *pi);

/* Replace α (host or device fp64 [C][D], all > 0) and the next EM-iteration index (resume /
 * single-step parity from an identical state). */
cmtcs_status cmtcs_set_state(cmtcs_ctx *ctx, const double *alpha, int32_t em_iter);

/* Probe-column CG transcripts of the last E-step (device buffers; NULL skips):
 *   gamma, xi fp64 [T_loc·C·K][cap] (NaN past steps), steps int32 [T_loc·C·K],
 *   mu_steps int32 [T_loc·C].  Column index (t·C + c)·K + k. */
cmtcs_status cmtcs_transcript(cmtcs_ctx *ctx, double *gamma, double *xi, int32_t *steps,
                              int32_t *mu_steps);

/* Message of the last failure on ctx (or of the last failed context-less call when ctx is NULL). */
const char *cmtcs_last_error(const cmtcs_ctx *ctx);
void cmtcs_destroy(cmtcs_ctx *ctx);

/* Total kernels this library launched on ctx since cmtcs_init (launch-count evidence). */
int64_t cmtcs_kernel_launches(const cmtcs_ctx *ctx);

/* Live device timing of em_step (enable = 0|1).  cmtcs_get_timing returns accumulated
 * milliseconds since the last reset (reset = 1 clears after reading):
 *   ms[0] operator phases (stages 1-2) of every CG step, ms[1] update phase (Alg. 1 lines 3-7):
 *         %globaltimer stamps taken inside the persistent CG kernel at its step boundaries;
 *   ms[2] everything in em_step after the CG kernel (estimators, M-step): CUDA events;
 *   ms[3] the whole persistent CG kernel: CUDA events recorded on the context's stream
 *         immediately before and after its launch;
 * n[0..1] CG steps, n[2..3] EM iterations. */
cmtcs_status cmtcs_set_timing(cmtcs_ctx *ctx, int32_t enable);
cmtcs_status cmtcs_get_timing(cmtcs_ctx *ctx, double ms[4], int64_t n[4], int32_t reset);

/* This rank's Eq. 4 sums of the last em_step, BEFORE the all-reduce (Alg. 2 lines
 * 14-15): out (host or device) fp64 [C·D + C + 1] = [den_cd = Σ_t q_tc(μ²_tcd + max(s_tcd, floor))
 * row-major | num_c = Σ_t q_tc | Σ_t log p(y_t|θ̂)], t over this rank's tasks.  Summing the
 * outputs of the ranks gives the all-reduced sums the M-step uses (multi-GPU tests).
 * ESTATE before any em_step. */
cmtcs_status cmtcs_estep_sums(cmtcs_ctx *ctx, double *out);

/* ---- stateless kernel entry points (unit tests / benchmarks; all pointers device) ------- */

/* Probe words (reading A6): out[(((i·C + c)·K + k)·nw + w] for local task i = 0..T_loc−1,
 * global task t0 + i, EM iteration `it`; nw = ceil(D/64). */
cmtcs_status cmtcs_probe_words(uint64_t seed, int32_t it, int32_t T, int32_t t0, int32_t T_loc,
                               int32_t C, int32_t K, int32_t D, uint64_t *out, void *cuda_stream);

/* Lanczos quadrature τ_j = D·Σ_u S̄²_{u,1} log λ̄_u of Γ̄(γ_j, ξ_j) (Eq. 7-8) for n columns:
 * gamma/xi fp64 [n][ld], steps int32 [n] (1 ≤ steps ≤ ld), tau fp64 [n].  scratch: fp64 of
 * 3·n·ld entries.  EEIG if any column fails. */
cmtcs_status cmtcs_lanczos_quadrature(const double *gamma, const double *xi, const int32_t *steps,
                                      int32_t n, int32_t ld, int32_t D, double *tau,
                                      double *scratch, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* CMTCS_H */
