// libcmtcs C ABI (include/cmtcs.h): context, workspace carving, the EM-iteration driver
// (Alg. 2 lines 2-16), NCCL all-reduce of the Eq. 4 sums, posterior readout.
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <new>

#include "cmtcs_internal.cuh"

using namespace cmtcs;

struct cmtcs_ctx {
  cmtcs_problem prob;
  double pi_host[MAXC];
  KParams kp;
  cudaStream_t stream;
  int device;
  int rank, world;
  ncclComm_t comm;
  bool have_comm;
  bool broken;
  bool have_estep;
  int em_iter;           // global index of the next EM iteration
  char err[512];
  double *h_out;         // pinned [32]: stats[16] | loglik | status(as int) ...
  int *h_status;         // pinned [8]
  int64_t launches;
  // live timing (cmtcs_set_timing)
  bool timing;
  cudaEvent_t tev[3];
  unsigned long long *h_ts;  // pinned [cap][4]
  double t_ms[4];
  int64_t t_n[4];
  // the CG loop: one persistent kernel per E-step (k_cg_persistent.cu), one CTA per SM
  TcMaps maps;
  int grid;
  int *h_u;                 // pinned: CG steps executed
  SimtTiming simt_tm;       // the FP32 engine's per-step events (created with the context)
  SimtStreams simt_ss;      // ... and its side stream for the mean columns
  bool have_simt_tm;
};

namespace {

thread_local char g_err[512];

cmtcs_status fail(cmtcs_ctx *c, cmtcs_status st, const char *fmt, ...) {
  char *buf = c ? c->err : g_err;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, 512, fmt, ap);
  va_end(ap);
  if (c && st != CMTCS_EINVAL) c->broken = true;
  return st;
}

#define CUDA_OK(ctx, call)                                                                    \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail((ctx), CMTCS_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                        \
  } while (0)

#define NCCL_OK(ctx, call)                                                                          \
  do {                                                                                              \
    ncclResult_t r_ = (call);                                                                       \
    if (r_ != ncclSuccess)                                                                          \
      return fail((ctx), CMTCS_ENCCL, "%s failed: %s", #call, ncclGetErrorString(r_));              \
  } while (0)

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Carver {
  char *base;
  size_t off = 0;
  template <class T>
  T *take(size_t n) {
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += align256(n * sizeof(T) + 1);
    return p;
  }
};

// widest column tile: 128 columns (TMEM holds the accumulators and the A stages; CMTCS_NTMAX
// overrides)
int nt_max(int shared_phi) {
  (void)shared_phi;
  const char *e = getenv("CMTCS_NTMAX");
  if (e) return std::max(16, std::min(TC_NTMAX, atoi(e) / 16 * 16));
  return TC_NTMAX;
}

TcCfg make_tc(const Dims &d) {
  TcCfg tc;
  tc.pair = d.pair;
  // a pair's MMA has N ≤ 256, a multiple of 32 (each CTA stages N/2 columns)
  tc.NT = std::min(nt_max(d.shared_phi), (d.P + (d.pair ? 31 : 15)) / (d.pair ? 32 : 16) * (d.pair ? 32 : 16));
  tc.slot = (tc.NT + 15) / 16 * 16;
  // TMEM (512 columns): accumulators in [0, acol0), the A stages (tf32 hi | lo, 64 columns) above:
  // three A stages with double-buffered accumulators when both fit, else two (CMTCS_SA overrides)
  tc.sa = 4 * tc.slot <= 512 - 64 * 3 ? 3 : 2;
  if (getenv("CMTCS_SA")) tc.sa = std::max(1, std::min(4, atoi(getenv("CMTCS_SA"))));
  tc.acol0 = 512 - 64 * tc.sa;
  tc.dbl = 4 * tc.slot <= tc.acol0 ? 1 : 0;
  tc.nacc = std::max(1, std::min(4, tc.acol0 / tc.slot - 1));   // main accumulators besides the cross one
  // ring stage: fp32 A (16 KB), B hi/lo (2 × NT × 128 B; a pair: its half, NT × 128 B), fp64
  // mean-column chunk (≤ 32 × Cp × 8 B)
  const unsigned mean_bytes = (256u * (unsigned)d.Cp + 1023u) & ~1023u;
  tc.stage_bytes = 128u * 128u + (tc.pair ? 1u : 2u) * (unsigned)tc.NT * 128u + mean_bytes;
  // one CTA per SM (512 TMEM columns) within ≤ 212 KB of the 227 KB of shared memory: the stage-2
  // epilogue's d tile (NT × 128 fp32) when ≥ 3 ring stages still fit (measured at C3: a 4th stage
  // instead of the d tile does not help, the K loop is bound by shared-memory traffic)
  const unsigned budget = 212u * 1024u;
  const unsigned dtile = (unsigned)tc.NT * 128u * 4u;
  int st_with = (int)((budget - std::min(budget, dtile)) / tc.stage_bytes);
  const int st_without = std::min(6, (int)(budget / tc.stage_bytes));
  if (getenv("CMTCS_NODTILE") ? atoi(getenv("CMTCS_NODTILE")) != 0 : tc.pair != 0) st_with = 0;   // pairs: ring stages, not the d tile
  if (st_with >= 3) {
    tc.use_dtile = 1;
    tc.dtile_bytes = dtile;
    tc.stages = std::min(6, st_with);
  } else {
    tc.use_dtile = 0;
    tc.dtile_bytes = 0;
    tc.stages = std::max(2, st_without);
  }
  return tc;
}

bool make_dims(const cmtcs_problem *p, Dims *d, char *why) {
  if (!p) { snprintf(why, 256, "problem is NULL"); return false; }
  if (p->T < 1 || p->N < 4 || p->D < 4 || p->C < 1 || p->K < 1) { snprintf(why, 256, "need T>=1, N>=4, D>=4, C>=1, K>=1"); return false; }
  if (p->N % 4 || p->D % 4) { snprintf(why, 256, "N and D must be multiples of 4 (got N=%d D=%d)", p->N, p->D); return false; }
  if (p->C > MAXC) { snprintf(why, 256, "C=%d exceeds the supported maximum %d", p->C, MAXC); return false; }
  if (!(p->beta > 0) || !std::isfinite(p->beta)) { snprintf(why, 256, "beta must be finite and > 0"); return false; }
  if (p->cg_max_iters < 1 || p->cg_max_iters > 12000) { snprintf(why, 256, "cg_max_iters must be in [1, 12000]"); return false; }
  if (!(p->cg_rel_tol >= 0)) { snprintf(why, 256, "cg_rel_tol must be >= 0"); return false; }
  if (!(p->alpha_max > 0) || !(p->var_floor >= 0) || !(p->empty_eps >= 0)) { snprintf(why, 256, "bad alpha_max/var_floor/empty_eps"); return false; }
  if (p->task_begin < 0 || p->task_end > p->T || p->task_end <= p->task_begin) { snprintf(why, 256, "bad task range [%d,%d) of T=%d", p->task_begin, p->task_end, p->T); return false; }
  if (p->em_iter0 < 0) { snprintf(why, 256, "em_iter0 must be >= 0"); return false; }
  if (!p->pi) { snprintf(why, 256, "pi is NULL"); return false; }
  double s = 0;
  for (int c = 0; c < p->C; ++c) {
    if (!(p->pi[c] > 0) || !std::isfinite(p->pi[c])) { snprintf(why, 256, "pi[%d] must be > 0", c); return false; }
    s += p->pi[c];
  }
  if (fabs(s - 1.0) > 1e-9) { snprintf(why, 256, "pi sums to %.17g, not 1", s); return false; }
  if (p->learn_pi != 0 && p->learn_pi != 1) { snprintf(why, 256, "learn_pi must be 0 or 1"); return false; }
  if (p->op_kind != CMTCS_OP_DENSE && p->op_kind != CMTCS_OP_PARTIAL_FOURIER && p->op_kind != CMTCS_OP_DENSE_FP32) {
    snprintf(why, 256, "unknown op_kind %d", p->op_kind);
    return false;
  }
  if (p->op_kind == CMTCS_OP_PARTIAL_FOURIER) {
    if (p->shared_phi) { snprintf(why, 256, "the partial-Fourier operator has a mask per task: shared_phi must be 0"); return false; }
    if (!p->fourier_rows) { snprintf(why, 256, "the partial-Fourier operator needs fourier_rows"); return false; }
    if (!fourier_supported(p->D, p->N, why)) return false;
  }
  d->T = p->T;
  d->Tl = p->task_end - p->task_begin;
  d->t0 = p->task_begin;
  d->N = p->N;
  d->D = p->D;
  d->C = p->C;
  d->K = p->K;
  d->P = p->C * p->K;
  d->Pp = (d->P + 3) & ~3;
  d->ldv = p->op_kind == CMTCS_OP_DENSE_FP32 ? (p->task_end - p->task_begin) * d->Pp : 0;
  d->Cp = (p->C + 1) & ~1;
  d->cap = p->cg_max_iters;
  d->nw = (p->D + 63) / 64;
  d->nRT1 = (p->N + OP_BR - 1) / OP_BR;
  d->nRT2 = (p->D + OP_BR - 1) / OP_BR;
  {
    // CTA pairs (2-CTA clusters, cta_group::2) when the operator has enough row-tile pairs to fill
    // the 74 pairs of a B200 twice over: half of B per CTA, M = 256 MMAs.  CMTCS_PAIR=0 disables,
    // =2 forces them (tests: every shape through the pair path)
    const char *e = getenv("CMTCS_PAIR");
    const int mode = p->op_kind != CMTCS_OP_DENSE ? 0 : e ? atoi(e) : 0;   // off by default: slower at C4 so far
    const int NT1 = std::min(nt_max(p->shared_phi), (d->P + 15) / 16 * 16);
    const long pair_units = (long)((d->P + NT1 - 1) / NT1) * ((d->nRT1 + 1) / 2) * (p->task_end - p->task_begin);
    d->pair = mode == 2 || (mode == 1 && pair_units >= 148);
  }
  const int NT = std::min(nt_max(p->shared_phi), (d->P + (d->pair ? 31 : 15)) / (d->pair ? 32 : 16) * (d->pair ? 32 : 16));   // = make_tc's NT
  d->nCT = (d->P + NT - 1) / NT;
  if (d->pair) {
    d->S1 = 1;
    d->K1 = (p->D + 31) / 32 * 32;
    d->split_coop = 0;
  } else {
    // split the stage-1 contraction over D (S1 ∈ {1, 2, 4, 8}, every split ≥ 128 of D) so that the
    // stage-1 units fill and balance the persistent grid (148 CTAs on a B200): minimise rounds ×
    // (chunks per unit + a fixed per-unit cost).  The split partial tiles are reduced cooperatively
    // when all stage-1 units fit in one round, else by the last-arriving split CTA
    // (k_cg_persistent.cu).
    const int sms = 148;
    const long base = (long)d->nCT * d->nRT1 * (p->task_end - p->task_begin);
    int best = 1;
    long best_cost = -1;
    for (int s1 = 1; s1 <= 8; s1 *= 2) {
      if (s1 > 1 && p->D / s1 < 128) break;
      const long rounds = (base * s1 + sms - 1) / sms;
      const long chunks = ((p->D + s1 - 1) / s1 + 31) / 32;
      const long cost = rounds * (chunks + 4);   // + fixed per-unit cost (prologue, epilogue, reduction)
      if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = s1; }
    }
    if (getenv("CMTCS_S1")) best = std::max(1, std::min(8, atoi(getenv("CMTCS_S1"))));   // experiments
    int k1 = (p->D + best - 1) / best;
    k1 = (k1 + 31) / 32 * 32;   // whole 32-wide K stages of the tensor-core pipeline
    d->K1 = k1;
    d->S1 = (p->D + k1 - 1) / k1;
    d->split_coop = d->S1 > 1 && base * d->S1 <= sms;
    if (d->S1 < 1 || d->S1 > 8) { snprintf(why, 256, "internal: bad split of D=%d", p->D); return false; }
  }
  d->shared_phi = p->shared_phi ? 1 : 0;
  d->phi_task_stride = p->shared_phi ? 0 : (int64_t)p->N * p->D;
  d->op = p->op_kind;
  if (d->op != CMTCS_OP_DENSE) d->pair = 0;   // the tensor-core operator only
  return true;
}

size_t carve(const Dims &d, char *base, Bufs *b) {
  Carver cv{base};
  const size_t Tl = d.Tl, P = d.P, C = d.C, D = d.D, N = d.N, cap = d.cap;
  b->alpha64 = cv.take<double>(C * D);
  b->alpha32 = cv.take<float>(C * D);
  b->logsum_alpha = cv.take<double>(C);
  b->logpi = cv.take<double>(C);
  b->b64 = cv.take<double>(Tl * D);
  b->bnorm2 = cv.take<double>(Tl);
  const size_t mats = d.shared_phi ? 1 : Tl;
  // dn = 0: the partial-Fourier operator keeps its CG vectors on chip (k_fourier.cu) — only x leaves;
  // tc = 0: the FP32 engine (k_simt.cu) has no tf32 pairs and no split-K partials
  const size_t dn = d.op == CMTCS_OP_PARTIAL_FOURIER ? 0 : 1;
  const size_t tc = d.op == CMTCS_OP_DENSE ? 1 : 0;
  b->PT = cv.take<float>(dn * mats * N * D);   // Φᵀ: both dense engines' M-major operand
  const size_t PV = d.ldv ? (size_t)d.Pp : P;   // FP32 engine: d-major with padded task blocks
  b->X = cv.take<float>(Tl * PV * D);
  b->R = cv.take<float>(dn * Tl * PV * D);
  b->D32 = cv.take<float>(dn * Tl * PV * D);
  b->Dh = cv.take<float>(tc * Tl * P * D);
  b->Dl = cv.take<float>(tc * Tl * P * D);
  b->W = cv.take<float>(dn * Tl * PV * D);
  b->Xm = cv.take<double>(Tl * C * D);
  b->Rm = cv.take<double>(dn * Tl * C * D);
  b->Dm = cv.take<double>(dn * Tl * C * D);
  b->Wm = cv.take<double>(dn * Tl * C * D);
  b->Uh = cv.take<float>(dn * Tl * d.Pp * N);
  b->Ul = cv.take<float>(tc * Tl * d.Pp * N);
  b->Um = cv.take<double>(dn * Tl * N * d.Cp);
  b->rr = cv.take<double>(Tl * P);
  b->rrm = cv.take<double>(Tl * C);
  b->dAd = cv.take<double>(dn * Tl * P * d.nRT2);
  b->dAdm = cv.take<double>(dn * Tl * C * d.nRT2);
  b->flag = cv.take<int>(Tl * P);
  b->flagm = cv.take<int>(Tl * C);
  b->steps = cv.take<int>(Tl * P);
  b->stepsm = cv.take<int>(Tl * C);
  b->act = cv.take<int>(Tl * P);
  b->m_act = cv.take<int>(Tl);
  b->gam = cv.take<double>(Tl * P * cap);
  b->xi = cv.take<double>(Tl * P * cap);
  b->tau = cv.take<double>(Tl * P);
  b->s = cv.take<double>(Tl * C * D);
  b->nu = cv.take<double>(Tl * C);
  b->ell = cv.take<double>(Tl * C);
  b->q = cv.take<double>(Tl * C);
  b->ll = cv.take<double>(Tl);
  b->red = cv.take<double>(C * D + C + 1);
  b->red_local = cv.take<double>(C * D + C + 1);
  b->alive = cv.take<int>(2 * cap);
  b->hist = cv.take<int>(cap);
  b->histm = cv.take<int>(cap);
  b->histt = cv.take<int>(cap);
  b->histp = cv.take<int>(cap);
  b->status = cv.take<int>(8);
  b->u = cv.take<int>(1);
  b->ts = cv.take<unsigned long long>((size_t)cap * 4 + 512);   // + 2 × 256 diagnostic stamps
  b->stats = cv.take<double>(16);
  b->assign = cv.take<int>(Tl);
  b->Upart = cv.take<float>(tc && d.S1 > 1 ? Tl * d.S1 * d.Pp * N : 1);
  b->Umpart = cv.take<double>(tc && d.S1 > 1 ? Tl * d.S1 * N * d.Cp : 1);
  b->resm = cv.take<double>(Tl * C);
  b->ftw = cv.take<double>(d.op == CMTCS_OP_PARTIAL_FOURIER ? 2 * D : 1);
  b->tmark = cv.take<int>(Tl);
  b->tilecnt = cv.take<int>(Tl * d.nCT * d.nRT1);
  b->gridbar = cv.take<unsigned>(1);
  b->dep = cv.take<int>(2 * Tl);
  if (!tc) b->Dh = b->Dl = b->Ul = nullptr;   // not carved: kernels must not touch them
  if (!dn) b->PT = nullptr;
  return cv.off;
}

__global__ void k_alpha_copy(double *a64, float *a32, double *logpi, const double *pi, int n, int C) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a32[i] = (float)a64[i];
  if (logpi && blockIdx.x == 0 && threadIdx.x < C) logpi[threadIdx.x] = log(pi[threadIdx.x]);
}

__global__ void k_check_alpha(const double *a, int n, int *bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (!(a[i] > 0.0) || !isfinite(a[i])) atomicExch(bad, 1);
}

cmtcs_status set_alpha(cmtcs_ctx *c, const double *alpha) {
  const Dims &d = c->kp.d;
  const size_t n = (size_t)d.C * d.D;
  // validated in scratch (red, rewritten by every M-step) so that a rejected α leaves the state intact
  CUDA_OK(c, cudaMemcpyAsync(c->kp.b.red, alpha, n * sizeof(double), cudaMemcpyDefault, c->stream));
  CUDA_OK(c, cudaMemsetAsync(c->kp.b.status + 4, 0, sizeof(int), c->stream));
  k_check_alpha<<<64, 256, 0, c->stream>>>(c->kp.b.red, (int)n, c->kp.b.status + 4);
  CUDA_OK(c, cudaMemcpyAsync(c->h_status + 4, c->kp.b.status + 4, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  if (c->h_status[4]) return fail(c, CMTCS_EINVAL, "alpha must be finite and > 0 everywhere");
  CUDA_OK(c, cudaMemcpyAsync(c->kp.b.alpha64, c->kp.b.red, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  k_alpha_copy<<<64, 256, 0, c->stream>>>(c->kp.b.alpha64, c->kp.b.alpha32, nullptr, nullptr, (int)n, d.C);
  CUDA_OK(c, cudaGetLastError());
  CUDA_OK(c, launch_alpha_stats(c->kp, c->stream));
  c->launches += 3;
  return CMTCS_OK;
}

const char *status_name(int code) {
  switch (code) {
    case ST_BREAKDOWN: return "CG breakdown (d'Ad <= 0)";
    case ST_EIG: return "Lanczos quadrature failed (eigen-iteration or Ritz value <= 0)";
    case ST_NUMERIC: return "non-finite ell / softmax of all -inf";
    default: return "unknown";
  }
}

cmtcs_status one_em_iteration(cmtcs_ctx *c, const uint64_t *probe_bits, const double *q_override,
                              cmtcs_step_info *info) {
  KParams kp = c->kp;
  const Dims &d = kp.d;
  cudaStream_t s = c->stream;
  kp.it = c->em_iter;
  kp.probe_bits = probe_bits;
  kp.q_override = q_override;
  int64_t L = 0;
  CUDA_OK(c, cudaMemsetAsync(kp.b.alive, 0, sizeof(int) * 2 * d.cap, s));
  CUDA_OK(c, cudaMemsetAsync(kp.b.hist, 0, sizeof(int) * d.cap, s));
  CUDA_OK(c, cudaMemsetAsync(kp.b.histm, 0, sizeof(int) * d.cap, s));
  CUDA_OK(c, cudaMemsetAsync(kp.b.histt, 0, sizeof(int) * d.cap, s));
  CUDA_OK(c, cudaMemsetAsync(kp.b.histp, 0, sizeof(int) * d.cap, s));
  CUDA_OK(c, cudaMemsetAsync(kp.b.tmark, 0, sizeof(int) * d.Tl, s));
  const bool fourier = d.op == CMTCS_OP_PARTIAL_FOURIER;
  if (fourier) {
    CUDA_OK(c, cudaMemsetAsync(kp.b.u, 0, sizeof(int), s));
  } else {
    CUDA_OK(c, launch_init_columns(kp, s));
    L += d.ldv ? 2 : 1;
  }
  const bool tm = c->timing;
  if (tm) {
    CUDA_OK(c, cudaMemsetAsync(kp.b.ts, 0, sizeof(unsigned long long) * (4 * d.cap + 256), s));
    CUDA_OK(c, cudaEventRecord(c->tev[0], s));
  }
  // ---- batched CG (Alg. 1) over all T_loc·C·(K+1) columns: one persistent kernel ----
  if (fourier) {
    CUDA_OK(c, launch_fourier_cg(kp, c->grid, s));   // probe columns (fp32), then mean columns (fp64)
  } else if (d.op == CMTCS_OP_DENSE_FP32) {
    c->simt_tm.op_ms = c->simt_tm.upd_ms = 0.0;
    CUDA_OK(c, run_simt_cg(kp, c->h_u, &L, tm ? &c->simt_tm : nullptr, c->simt_ss, s));   // L counts the per-step kernels
  } else {
    CUDA_OK(c, launch_cg_persistent(kp, c->maps, c->grid, s));
  }
  if (tm) CUDA_OK(c, cudaEventRecord(c->tev[1], s));
  // ---- estimators: s (Eq. 5), ν̄ (Eq. 7-9), Φμ for ℓ, q and log-lik (Eq. 3) ----
  CUDA_OK(c, launch_diag(kp, s));
  CUDA_OK(c, launch_lanczos(kp.b.gam, kp.b.xi, kp.b.steps, d.Tl * d.P, d.cap, d.D, kp.b.tau, nullptr,
                            kp.b.status, s));
  if (!fourier) CUDA_OK(c, launch_mu_stage1(kp, kp.b.Xm, s));   // Φμ (the Fourier kernel forms ‖y − Φμ‖² itself)
  CUDA_OK(c, launch_estep_finish(kp, s));
  // ---- M-step (Eq. 4): local sums → all-reduce over ranks → α update ----
  CUDA_OK(c, launch_mstep_partial(kp, s));
  L += 5;
  // this rank's Eq. 4 sums before the all-reduce (cmtcs_estep_sums)
  CUDA_OK(c, cudaMemcpyAsync(kp.b.red_local, kp.b.red, sizeof(double) * ((size_t)d.C * d.D + d.C + 1),
                             cudaMemcpyDeviceToDevice, s));
  if (c->have_comm)
    NCCL_OK(c, ncclAllReduce(kp.b.red, kp.b.red, (size_t)d.C * d.D + d.C + 1, ncclDouble, ncclSum, c->comm, s));
  CUDA_OK(c, launch_mstep_finish(kp, s));
  CUDA_OK(c, launch_alpha_stats(kp, s));
  {
    const size_t n = (size_t)d.C * d.D;
    k_alpha_copy<<<64, 256, 0, s>>>(kp.b.alpha64, kp.b.alpha32, nullptr, nullptr, (int)n, d.C);
    CUDA_OK(c, cudaGetLastError());
  }
  CUDA_OK(c, launch_stats(kp, s));
  L += 4;
  if (tm) {
    CUDA_OK(c, cudaEventRecord(c->tev[2], s));
    CUDA_OK(c, cudaMemcpyAsync(c->h_ts, kp.b.ts, sizeof(unsigned long long) * (4 * d.cap + 512), cudaMemcpyDeviceToHost, s));
  }
  CUDA_OK(c, cudaMemcpyAsync(c->h_u, kp.b.u, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_OK(c, cudaMemcpyAsync(c->h_out, kp.b.stats, 16 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_OK(c, cudaMemcpyAsync(c->h_out + 16, kp.b.red + (size_t)d.C * d.D + d.C, sizeof(double),
                             cudaMemcpyDeviceToHost, s));
  CUDA_OK(c, cudaMemcpyAsync(c->h_status, kp.b.status, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_OK(c, cudaStreamSynchronize(s));
  c->launches += L;
  c->have_estep = true;
  const int steps_run = *c->h_u;
  const int cg_k = fourier ? 2 : d.op == CMTCS_OP_DENSE ? 1 : 0;   // the persistent CG kernel (partial
  L += cg_k;                                                          // Fourier: probe and mean kernels)
  c->launches += cg_k;
  if (tm) {
    // per CG step: %globaltimer stamps taken by CTA 0 after the grid barriers: step start,
    // operator (phases 1-2) done, update (phase 3) done (device clock, ns)
    if (d.op == CMTCS_OP_DENSE_FP32) {   // CUDA events around the operator and update kernels
      c->t_ms[0] += c->simt_tm.op_ms;
      c->t_ms[1] += c->simt_tm.upd_ms;
    }
    for (int u = 0; u < steps_run && d.op != CMTCS_OP_DENSE_FP32; ++u) {
      const unsigned long long *q = c->h_ts + 4 * u;
      const unsigned long long t0 = q[0], t1 = q[1], t2 = q[2];
      if (t0 && t1 >= t0) c->t_ms[0] += (t1 - t0) * 1e-6;
      if (t1 && t2 >= t1) c->t_ms[1] += (t2 - t1) * 1e-6;
    }
    if (getenv("CMTCS_PHASE_LOG") && steps_run > 0) {   // diagnostic: mean per-step phase durations (device stamps)
      double ph[3] = {0, 0, 0};
      for (int u = 0; u < steps_run; ++u) {
        const unsigned long long *q = c->h_ts + 4 * u;
        ph[0] += (q[3] - q[0]) * 1e-3;
        ph[1] += (q[1] - q[3]) * 1e-3;
        ph[2] += (q[2] - q[1]) * 1e-3;
      }
      fprintf(stderr, "[cmtcs] EM it %d: %d CG steps, per step us: phase1 %.2f phase2 %.2f update %.2f\n",
              c->em_iter, steps_run, ph[0] / steps_run, ph[1] / steps_run, ph[2] / steps_run);
      for (int ph = 0; ph < 2 && steps_run > c->kp.trace_step; ++ph) {
        const unsigned long long *g = c->h_ts + 4 * d.cap + 256 * ph;
        const unsigned long long t0 = g[127];   // SM clock at the phase start (CTA 0)
        auto us = [&](int i) { return g[i] ? ((double)g[i] - (double)t0) * 1e-3 : -1.0; };
        fprintf(stderr, "[cmtcs]   phase %d CTA0 unit0 (kilocycles): prod start %.2f epi start %.2f\n", ph + 1, us(84), us(83));
        fprintf(stderr, "[cmtcs]     prod acq :"); for (int i = 0; i < 16; ++i) fprintf(stderr, " %.2f", us(i));
        fprintf(stderr, "\n[cmtcs]     prod iss :"); for (int i = 16; i < 32; ++i) fprintf(stderr, " %.2f", us(i));
        fprintf(stderr, "\n[cmtcs]     mma full :"); for (int i = 32; i < 48; ++i) fprintf(stderr, " %.2f", us(i));
        fprintf(stderr, "\n[cmtcs]     A full   :"); for (int i = 48; i < 64; ++i) fprintf(stderr, " %.2f", us(i));
        fprintf(stderr, "\n[cmtcs]     A aempty :"); for (int i = 64; i < 80; ++i) fprintf(stderr, " %.2f", us(i));
        fprintf(stderr, "\n[cmtcs]     A split  :"); for (int i = 90; i < 106; ++i) fprintf(stderr, " %.2f", us(i));
        fprintf(stderr, "\n[cmtcs]     A done   :"); for (int i = 106; i < 120; ++i) fprintf(stderr, " %.2f", us(i));
        fprintf(stderr, "\n[cmtcs]     epi grp  :"); for (int i = 128; i < 160; ++i) fprintf(stderr, " %.2f", us(i));
        if (ph == 1) {
          for (int q = 0; q < 4; ++q) { fprintf(stderr, "\n[cmtcs]     afull q%d :", q); for (int i = 0; i < 16; ++i) fprintf(stderr, " %.2f", us(160 + 16 * q + i)); }
          fprintf(stderr, "\n[cmtcs]     mfull    :"); for (int i = 0; i < 16; ++i) fprintf(stderr, " %.2f", us(240 + i));
          fprintf(stderr, "\n[cmtcs]     mdone    :"); for (int i = 0; i < 16; ++i) fprintf(stderr, " %.2f", us(224 + i));
        }
        if (ph == 0) { fprintf(stderr, "\n[cmtcs]     update (kcyc from phase start): start %.2f gam %.2f pass1 %.2f xi %.2f end %.2f", (g[160]-g[168])*1e-3, (g[161]-g[168])*1e-3, (g[162]-g[168])*1e-3, (g[163]-g[168])*1e-3, (g[164]-g[168])*1e-3); }
        fprintf(stderr, "\n[cmtcs]     epi loopend %.2f meanepi %.2f tfull %.2f drained %.2f handoff %.2f end %.2f\n", us(85), us(86), us(80), us(81), us(87), us(82));

      }
    }
    float ms = 0.f, mk = 0.f;
    CUDA_OK(c, cudaEventElapsedTime(&ms, c->tev[1], c->tev[2]));
    CUDA_OK(c, cudaEventElapsedTime(&mk, c->tev[0], c->tev[1]));
    c->t_ms[2] += ms;
    c->t_ms[3] += mk;
    c->t_n[0] += steps_run;
    c->t_n[1] += steps_run;
    c->t_n[2] += 1;
    c->t_n[3] += 1;
  }
  const int it = c->em_iter;
  c->em_iter += 1;
  if (c->h_status[0] != ST_OK) {
    const int code = c->h_status[0];
    const cmtcs_status st = code == ST_BREAKDOWN ? CMTCS_EBREAKDOWN : code == ST_EIG ? CMTCS_EEIG : CMTCS_ENUMERIC;
    return fail(c, st, "EM iteration %d: %s at (task %d, column %d, step %d)", it, status_name(code),
                c->h_status[1], c->h_status[2], c->h_status[3]);
  }
  if (info) {
    const double *o = c->h_out;
    info->loglik = o[16] / (double)d.T;
    info->em_iter = it;
    info->cg_iters = (int32_t)std::max(o[1], o[4]);
    info->probe_steps_min = (int32_t)o[0];
    info->probe_steps_max = (int32_t)o[1];
    info->probe_steps_mean = o[2];
    info->mu_steps_min = (int32_t)o[3];
    info->mu_steps_max = (int32_t)o[4];
    info->n_cap_hit = (int64_t)o[5];
    info->probe_col_iters = (int64_t)o[6];
    info->mean_col_iters = (int64_t)o[7];
    info->task_iters = (int64_t)o[8];
    info->tile_col_iters = (int64_t)o[9];
    info->kernel_launches = L;
  }
  return CMTCS_OK;
}

}  // namespace

extern "C" {

cmtcs_status cmtcs_get_unique_id(uint8_t out[128]) {
  if (!out) return fail(nullptr, CMTCS_EINVAL, "out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, CMTCS_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  memcpy(out, &id, 128);
  return CMTCS_OK;
}

cmtcs_status cmtcs_workspace_size(const cmtcs_problem *p, size_t *bytes) {
  Dims d;
  char why[256];
  if (!bytes) return fail(nullptr, CMTCS_EINVAL, "bytes is NULL");
  if (!make_dims(p, &d, why)) return fail(nullptr, CMTCS_EINVAL, "%s", why);
  Bufs b;
  *bytes = carve(d, nullptr, &b);
  return CMTCS_OK;
}

cmtcs_status cmtcs_init(cmtcs_ctx **out, const cmtcs_problem *p, const float *phi, const float *y,
                        const double *alpha0, void *workspace, size_t workspace_bytes,
                        const uint8_t *nccl_uid, int32_t rank, int32_t world, int32_t device,
                        void *cuda_stream) {
  if (!out) return fail(nullptr, CMTCS_EINVAL, "ctx out-pointer is NULL");
  *out = nullptr;
  Dims d;
  char why[256];
  if (!make_dims(p, &d, why)) return fail(nullptr, CMTCS_EINVAL, "%s", why);
  const bool fourier = p->op_kind == CMTCS_OP_PARTIAL_FOURIER;
  if (fourier ? phi != nullptr : !phi) return fail(nullptr, CMTCS_EINVAL, fourier ? "phi must be NULL for the partial-Fourier operator" : "phi must be non-NULL");
  if (!y || !alpha0 || !workspace) return fail(nullptr, CMTCS_EINVAL, "y, alpha0 and workspace must be non-NULL");
  if (((uintptr_t)workspace & 255) || ((uintptr_t)phi & 15) || ((uintptr_t)y & 3))
    return fail(nullptr, CMTCS_EINVAL, "workspace must be 256-byte and phi 16-byte aligned");
  if (world < 1 || rank < 0 || rank >= world) return fail(nullptr, CMTCS_EINVAL, "bad rank %d / world %d", rank, world);
  if (world > 1 && !nccl_uid) return fail(nullptr, CMTCS_EINVAL, "world > 1 needs an NCCL unique id");
  Bufs b;
  const size_t need = carve(d, nullptr, &b);
  if (workspace_bytes < need) return fail(nullptr, CMTCS_ENOMEM, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(nullptr, CMTCS_ECUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  cmtcs_ctx *c = new (std::nothrow) cmtcs_ctx();
  if (!c) return fail(nullptr, CMTCS_ENOMEM, "host allocation failed");
  c->prob = *p;
  for (int i = 0; i < p->C; ++i) c->pi_host[i] = p->pi[i];
  c->prob.pi = c->pi_host;
  c->stream = (cudaStream_t)cuda_stream;
  c->device = device;
  c->rank = rank;
  c->world = world;
  c->em_iter = p->em_iter0;
  carve(d, (char *)workspace, &b);
  c->kp.d = d;
  c->kp.b = b;
  c->kp.tc = make_tc(d);
  c->kp.tc.pf = getenv("CMTCS_PF") ? atoi(getenv("CMTCS_PF")) : 0;
  c->kp.tc.l2hint = getenv("CMTCS_L2HINT") ? atoi(getenv("CMTCS_L2HINT")) : 0;
  c->kp.phi = phi;
  c->kp.y = y;
  c->kp.beta = p->beta;
  c->kp.learn_pi = p->learn_pi;
  c->kp.toff = c->kp.tcnt = 0;
  c->kp.tol = p->cg_rel_tol;
  c->kp.tol_mean = p->mean_rel_tol < 0 ? p->cg_rel_tol : p->mean_rel_tol;
  c->kp.alpha_max = p->alpha_max;
  c->kp.var_floor = p->var_floor;
  c->kp.empty_eps = p->empty_eps;
  c->kp.seed = p->probe_seed;
  c->kp.dbg_flags = getenv("CMTCS_DBG") ? atoi(getenv("CMTCS_DBG")) : 0;
  c->kp.trace_step = getenv("CMTCS_TRACE_STEP") ? atoi(getenv("CMTCS_TRACE_STEP")) : 5;
  *out = c;  // from here on errors leave a (broken) ctx the caller destroys
  CUDA_OK(c, cudaMallocHost((void **)&c->h_out, 32 * sizeof(double)));
  CUDA_OK(c, cudaMallocHost((void **)&c->h_status, 8 * sizeof(int)));

  CUDA_OK(c, cudaMallocHost((void **)&c->h_u, 2 * sizeof(int)));
  CUDA_OK(c, cudaMallocHost((void **)&c->h_ts, sizeof(unsigned long long) * (4 * d.cap + 512)));
  for (int i = 0; i < 3; ++i) CUDA_OK(c, cudaEventCreate(&c->tev[i]));
  if (p->op_kind == CMTCS_OP_DENSE_FP32) {
    for (int i = 0; i < 3 * SimtTiming::B; ++i) CUDA_OK(c, cudaEventCreate(&c->simt_tm.ev[i]));
    c->have_simt_tm = true;
    CUDA_OK(c, cudaStreamCreateWithFlags(&c->simt_ss.side, cudaStreamNonBlocking));
    CUDA_OK(c, cudaEventCreateWithFlags(&c->simt_ss.fork, cudaEventDisableTiming));
    CUDA_OK(c, cudaEventCreateWithFlags(&c->simt_ss.join, cudaEventDisableTiming));
  }
  CUDA_OK(c, cudaMemsetAsync(b.status, 0, 8 * sizeof(int), c->stream));
  CUDA_OK(c, cudaMemsetAsync(b.gam, 0, sizeof(double) * d.Tl * d.P * d.cap, c->stream));
  CUDA_OK(c, cudaMemsetAsync(b.xi, 0, sizeof(double) * d.Tl * d.P * d.cap, c->stream));
  c->kp.rows = p->fourier_rows;
  if (fourier) {
    int dev = 0;
    CUDA_OK(c, cudaGetDevice(&dev));
    CUDA_OK(c, cudaDeviceGetAttribute(&c->grid, cudaDevAttrMultiProcessorCount, dev));
  } else {
    CUDA_OK(c, cudaMemsetAsync(b.Um, 0, sizeof(double) * (size_t)d.Tl * d.N * d.Cp, c->stream));
    // U's padding rows P..Pp−1 of each task are B-tile rows past the tile's columns: keep them finite
    CUDA_OK(c, cudaMemsetAsync(b.Uh, 0, sizeof(float) * (size_t)d.Tl * d.Pp * d.N, c->stream));
    if (b.Ul) CUDA_OK(c, cudaMemsetAsync(b.Ul, 0, sizeof(float) * (size_t)d.Tl * d.Pp * d.N, c->stream));
  }
  if (p->op_kind == CMTCS_OP_DENSE) {   // the persistent tensor-core kernel
    CUDA_OK(c, cudaMemsetAsync(b.tilecnt, 0, sizeof(int) * d.Tl * d.nCT * d.nRT1, c->stream));
    c->grid = cg_grid_size(c->kp);
    if (c->grid < 1) return fail(c, CMTCS_ECUDA, "persistent CG kernel cannot be made resident (smem %zu bytes)",
                                 tc_smem_bytes(c->kp.tc, d.P));
    if (d.split_coop && (long)d.Tl * d.nCT * d.nRT1 * d.S1 > c->grid)
      return fail(c, CMTCS_ECUDA, "cooperative split-K needs all %d stage-1 units co-resident but the grid has %d CTAs",
                  d.Tl * d.nCT * d.nRT1 * d.S1, c->grid);
  }
  // π: log π_c on device
  double *pi_dev = b.red;  // scratch: red is rewritten every M-step
  CUDA_OK(c, cudaMemcpyAsync(pi_dev, c->pi_host, sizeof(double) * p->C, cudaMemcpyHostToDevice, c->stream));
  k_alpha_copy<<<1, 32, 0, c->stream>>>(b.alpha64, b.alpha32, b.logpi, pi_dev, 0, p->C);
  CUDA_OK(c, cudaGetLastError());
  cmtcs_status st = set_alpha(c, alpha0);
  if (st != CMTCS_OK) { c->broken = true; return st; }
  if (fourier) {
    CUDA_OK(c, launch_fourier_rhs(c->kp, c->stream));
    c->launches += 3;
  } else {
    CUDA_OK(c, launch_rhs(c->kp, c->stream));
    CUDA_OK(c, launch_split_phi(c->kp, c->stream));   // Φᵀ
    c->launches += 3;
    if (p->op_kind == CMTCS_OP_DENSE) {
      c->launches += 1;
      char why[256];
      if (!encode_maps(c->kp, &c->maps, why)) return fail(c, CMTCS_ECUDA, "%s", why);
    }
  }
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  if (world > 1 || nccl_uid) {   // a uid with world == 1: a 1-rank communicator (the NCCL path on one GPU)
    ncclUniqueId id;
    memcpy(&id, nccl_uid, 128);
    NCCL_OK(c, ncclCommInitRank(&c->comm, world, id, rank));
    c->have_comm = true;
  }
  return CMTCS_OK;
}

cmtcs_status cmtcs_em_step(cmtcs_ctx *c, int32_t n_iters, const uint64_t *probe_bits,
                           const double *q_override, cmtcs_step_info *info) {
  if (!c) return fail(nullptr, CMTCS_EINVAL, "ctx is NULL");
  if (c->broken) return CMTCS_ESTATE;
  if (n_iters < 1) return fail(c, CMTCS_EINVAL, "n_iters must be >= 1");
  if ((probe_bits || q_override) && n_iters != 1)
    return fail(c, CMTCS_EINVAL, "probe_bits / q_override require n_iters == 1");
  CUDA_OK(c, cudaSetDevice(c->device));
  for (int i = 0; i < n_iters; ++i) {
    cmtcs_status st = one_em_iteration(c, probe_bits, q_override, info);
    if (st != CMTCS_OK) return st;
  }
  return CMTCS_OK;
}

cmtcs_status cmtcs_posterior(cmtcs_ctx *c, double *mu, double *s, double *logdet, double *q,
                             double *alpha, int32_t *assign, double *recon) {
  if (!c) return fail(nullptr, CMTCS_EINVAL, "ctx is NULL");
  if (c->broken) return CMTCS_ESTATE;
  if (!c->have_estep) return fail(c, CMTCS_ESTATE, "posterior requested before any em_step");
  const Dims &d = c->kp.d;
  const Bufs &b = c->kp.b;
  cudaStream_t st = c->stream;
  const size_t tcd = (size_t)d.Tl * d.C * d.D, tc = (size_t)d.Tl * d.C;
  if (mu) CUDA_OK(c, cudaMemcpyAsync(mu, b.Xm, tcd * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (s) CUDA_OK(c, cudaMemcpyAsync(s, b.s, tcd * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (logdet) CUDA_OK(c, cudaMemcpyAsync(logdet, b.nu, tc * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (q) CUDA_OK(c, cudaMemcpyAsync(q, b.q, tc * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (alpha) CUDA_OK(c, cudaMemcpyAsync(alpha, b.alpha64, (size_t)d.C * d.D * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (assign || recon) {
    CUDA_OK(c, launch_readout(c->kp, recon, st));
    c->launches += 1;
    if (assign) CUDA_OK(c, cudaMemcpyAsync(assign, b.assign, d.Tl * sizeof(int), cudaMemcpyDeviceToDevice, st));
  }
  return CMTCS_OK;
}

cmtcs_status cmtcs_get_pi(cmtcs_ctx *c, double *pi) {
  if (!c) return fail(nullptr, CMTCS_EINVAL, "ctx is NULL");
  if (c->broken) return CMTCS_ESTATE;
  if (!pi) return fail(c, CMTCS_EINVAL, "pi is NULL");
  const int C = c->kp.d.C;
  double lp[MAXC], v[MAXC];
  CUDA_OK(c, cudaMemcpyAsync(lp, c->kp.b.logpi, C * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  for (int i = 0; i < C; ++i) v[i] = exp(lp[i]);
  CUDA_OK(c, cudaMemcpy(pi, v, C * sizeof(double), cudaMemcpyDefault));
  return CMTCS_OK;
}

cmtcs_status cmtcs_set_state(cmtcs_ctx *c, const double *alpha, int32_t em_iter) {
  if (!c) return fail(nullptr, CMTCS_EINVAL, "ctx is NULL");
  if (c->broken) return CMTCS_ESTATE;
  if (em_iter < 0) return fail(c, CMTCS_EINVAL, "em_iter must be >= 0");
  if (alpha) {
    cmtcs_status st = set_alpha(c, alpha);
    if (st != CMTCS_OK) return st;
  }
  c->em_iter = em_iter;
  return CMTCS_OK;
}

cmtcs_status cmtcs_transcript(cmtcs_ctx *c, double *gamma, double *xi, int32_t *steps, int32_t *mu_steps) {
  if (!c) return fail(nullptr, CMTCS_EINVAL, "ctx is NULL");
  if (c->broken) return CMTCS_ESTATE;
  if (!c->have_estep) return fail(c, CMTCS_ESTATE, "transcript requested before any em_step");
  const Dims &d = c->kp.d;
  if (gamma || xi) {
    CUDA_OK(c, launch_copy_transcript(c->kp, gamma, xi, c->stream));
    c->launches += 1;
  }
  if (steps) CUDA_OK(c, cudaMemcpyAsync(steps, c->kp.b.steps, sizeof(int) * d.Tl * d.P, cudaMemcpyDeviceToDevice, c->stream));
  if (mu_steps) CUDA_OK(c, cudaMemcpyAsync(mu_steps, c->kp.b.stepsm, sizeof(int) * d.Tl * d.C, cudaMemcpyDeviceToDevice, c->stream));
  return CMTCS_OK;
}

cmtcs_status cmtcs_estep_sums(cmtcs_ctx *c, double *out) {
  if (!c || !out) return fail(c, CMTCS_EINVAL, "ctx and out must be non-NULL");
  if (c->broken) return CMTCS_ESTATE;
  if (!c->have_estep) return fail(c, CMTCS_ESTATE, "E-step sums requested before any em_step");
  const Dims &d = c->kp.d;
  CUDA_OK(c, cudaMemcpyAsync(out, c->kp.b.red_local, sizeof(double) * ((size_t)d.C * d.D + d.C + 1),
                             cudaMemcpyDefault, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  return CMTCS_OK;
}

const char *cmtcs_last_error(const cmtcs_ctx *c) { return c ? c->err : g_err; }

void cmtcs_destroy(cmtcs_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->have_comm) ncclCommDestroy(c->comm);

  for (int i = 0; i < 3; ++i)
    if (c->tev[i]) cudaEventDestroy(c->tev[i]);
  if (c->have_simt_tm) {
    for (int i = 0; i < 3 * SimtTiming::B; ++i)
      if (c->simt_tm.ev[i]) cudaEventDestroy(c->simt_tm.ev[i]);
    if (c->simt_ss.side) {
      cudaStreamSynchronize(c->simt_ss.side);
      cudaStreamDestroy(c->simt_ss.side);
    }
    if (c->simt_ss.fork) cudaEventDestroy(c->simt_ss.fork);
    if (c->simt_ss.join) cudaEventDestroy(c->simt_ss.join);
  }
  if (c->h_u) cudaFreeHost(c->h_u);
  if (c->h_ts) cudaFreeHost(c->h_ts);
  if (c->h_out) cudaFreeHost(c->h_out);
  if (c->h_status) cudaFreeHost(c->h_status);
  delete c;
}

int64_t cmtcs_kernel_launches(const cmtcs_ctx *c) { return c ? c->launches : 0; }

cmtcs_status cmtcs_set_timing(cmtcs_ctx *c, int32_t enable) {
  if (!c) return fail(nullptr, CMTCS_EINVAL, "ctx is NULL");
  if (c->broken) return CMTCS_ESTATE;
  c->timing = enable != 0;
  return CMTCS_OK;
}

cmtcs_status cmtcs_get_timing(cmtcs_ctx *c, double ms[4], int64_t n[4], int32_t reset) {
  if (!c) return fail(nullptr, CMTCS_EINVAL, "ctx is NULL");
  for (int i = 0; i < 4; ++i) {
    if (ms) ms[i] = c->t_ms[i];
    if (n) n[i] = c->t_n[i];
    if (reset) { c->t_ms[i] = 0; c->t_n[i] = 0; }
  }
  return CMTCS_OK;
}

cmtcs_status cmtcs_probe_words(uint64_t seed, int32_t it, int32_t T, int32_t t0, int32_t T_loc, int32_t C,
                               int32_t K, int32_t D, uint64_t *out, void *stream) {
  if (!out || T < 1 || t0 < 0 || T_loc < 1 || t0 + T_loc > T || C < 1 || K < 1 || D < 1 || it < 0)
    return fail(nullptr, CMTCS_EINVAL, "bad arguments to cmtcs_probe_words");
  cudaError_t e = launch_probe_words(seed, it, T, t0, T_loc, C, K, D, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(nullptr, CMTCS_ECUDA, "probe words: %s", cudaGetErrorString(e));
  return CMTCS_OK;
}

cmtcs_status cmtcs_lanczos_quadrature(const double *gamma, const double *xi, const int32_t *steps, int32_t n,
                                      int32_t ld, int32_t D, double *tau, double *scratch, void *stream) {
  if (!gamma || !xi || !steps || !tau || !scratch || n < 0 || ld < 1 || D < 1)
    return fail(nullptr, CMTCS_EINVAL, "bad arguments to cmtcs_lanczos_quadrature");
  int *status = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMallocAsync((void **)&status, 8 * sizeof(int), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(status, 0, 8 * sizeof(int), s);
  if (e == cudaSuccess) e = launch_lanczos(gamma, xi, steps, n, ld, D, tau, scratch, status, s);
  int h[4] = {0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, status, 4 * sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (status) cudaFreeAsync(status, s);
  if (e != cudaSuccess) return fail(nullptr, CMTCS_ECUDA, "lanczos quadrature: %s", cudaGetErrorString(e));
  if (h[0] != ST_OK) return fail(nullptr, CMTCS_EEIG, "lanczos quadrature failed at column %d (%d, %d)", h[1], h[2], h[3]);
  return CMTCS_OK;
}

}  // extern "C"
