#!/usr/bin/env python
"""bench.py — throughput of the CoFEM hot path (EM iterations/s of the T×C×(K+1) batched-CG E-step
plus M-step) on N B200s, and of the fp64 CPU oracle as the reference arm.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl cuda|reference]

A "step" is one EM iteration (Alg. 2 lines 2-16) over the whole workload of
BASELINE.json configs[cfg-1] (default configs[3] = C4, the metric's multi-GPU scaling config and
the largest per-task config that fits one GPU), continuing the EM run: W untimed warm-up
iterations, then K timed ones.  For N > 1 (torchrun, one rank per GPU, NCCL) the config's T tasks
are sharded in contiguous blocks (--scaling strong, the default: `value` is EM iterations/s of the
configured problem) and the M-step sums are all-reduced inside libcmtcs (the method's one exchange
step).  --scaling weak instead gives every rank a config-sized block (T_total = N·T) and reports
the job's throughput in config-sized EM iterations/s (EM iterations/s × N), labelled as such.
Rank 0 prints one JSON line.  See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthetic  # noqa: E402

SM_COUNT = 148
FP32_LANES_PER_SM = 128
SM_MAX_MHZ = 1965.0


def baseline_json():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": SM_MAX_MHZ}, "fallback"


def fp32_peak_tflops(sm_mhz):
    """FFMA peak: 148 SMs × 128 FP32 lanes × 2 flop × clock (B200_PROFILING.md unit counts)."""
    return SM_COUNT * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12


def tf32x3_peak_tflops(peaks):
    """fp32-equivalent peak of the 3xTF32 tensor-core operator: measured dense bf16 × (tf32/bf16 =
    1.1/2.25 nominal, B200_PROFILING.md) ÷ 3 MMAs per product.  Burst figure: the operator kernels
    are timed individually (device stamps), sustained is reported alongside."""
    ratio = 1.1 / 2.25
    return peaks["bf16_tflops"] * ratio / 3.0, peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * ratio / 3.0


# north_star: "Tensor cores (3xTF32 split) are used only for the shared-Φ dense-contraction config,
# and only if the oracle tolerance holds".  Measured (tests/test_gpu_midrun.py): the
# tensor-core engine misses |ΔL| ≤ 1e-3 at C4 and C5 (truncating accumulation), C5 included; the FP32
# engine meets every bar everywhere.  auto = the FP32 engine at every dense config (reading E1).
def resolve_engine(name, cfg):
    if cfg.operator == "fourier":
        return "fourier"
    return "fp32" if name == "auto" else name


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5, 6],
                    help="BASELINE.json configs[cfg-1] (1-5); 6 = the paper's own partial-Fourier workload (§4)")
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle sample budget")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="EM iterations of the end-to-end leg (init from host buffers + steps + readback); 0 = all K")
    ap.add_argument("--engine", default="auto", choices=["auto", "tensor", "fp32"],
                    help="dense operator: FP32 CUDA cores or tcgen05 3xTF32 tensor cores; auto = the north_star's "
                         "rule (tensor cores only where the oracle tolerance holds: nowhere at C4/C5, so FP32; DESIGN.md §3 E1)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N > 1: strong = the config's tasks sharded (default), weak = a config-sized block per rank")
    return ap.parse_args()


# --------------------------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# --------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# --------------------------------------------------------------------------------------------
def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        if th:
            return int(max(th))
    except Exception:
        pass
    return os.cpu_count()


def oracle_blocks(cfg, alpha, it, budget_s):
    """Times the oracle (fp64 cofem, as it stands) on (task, cluster) blocks of EM iteration `it` at
    the state `alpha` — Alg. 2 lines 6-9 per block, the blocks of an E-step being
    independent — adding blocks in (task, cluster) order until `budget_s` of CPU work is spent.
    Returns (seconds per block, blocks done, CG steps of the sample)."""
    from oracle import cofem as O
    n, spent, steps = 0, 0.0, []
    data = None
    while n < cfg.T * cfg.C and spent < budget_s:
        t, c = divmod(n, cfg.C)
        if c == 0 or data is None:
            data = synthetic.generate(cfg, [t])
        if cfg.operator == "fourier":
            phi_t = O.partial_fourier_matrix(cfg.D, data["rows"][0])
        else:
            phi_t = data["phi"] if cfg.shared_phi else data["phi"][0]
        t0 = time.perf_counter()
        P = O.probe_signs(cfg.probe_seed, it, cfg.T, t, cfg.C, cfg.K, cfg.D)
        o = O.cofem_task(phi_t, data["y"][0], data["beta"], alpha, data["pi"], P, cfg.cg_tol, cfg.cg_cap,
                         clusters=[c])
        spent += time.perf_counter() - t0
        steps.append(int(np.max(o["probe_steps"])))
        n += 1
    return spent / n, n, steps


def cpu_baseline(cfg, budget_s, alpha, it):
    per_block, n, steps = oracle_blocks(cfg, alpha, it, budget_s)
    nblk = cfg.T * cfg.C
    return {"value": 1.0 / (per_block * nblk), "unit": "EM iters/s", "cores": cpu_cores(),
            "kind": "oracle",
            "sample": (f"oracle (numpy fp64, cofem mode) E-step blocks (task, cluster) of EM iteration {it} "
                       f"from the GPU arm's entry state of its first timed iteration: {n} of {nblk} blocks "
                       f"({per_block * n:.1f} s, max CG steps {max(steps)}), time x{nblk / n:.0f} to the full "
                       f"E-step; the M-step (< 0.1 % of the work) is not timed")}


def reference_arm(args):
    """The reference arm of this tier: the fp64 oracle, as it stands, on the host cores.  Each step
    is one EM iteration of a bounded sample of the workload — the first task's first `nc`
    clusters (each (t, c) block of Alg. 2 lines 6-9 is independent), EM continued on that sample
    with its own M-step — and `value` extrapolates the measured sample time to the configured
    workload (× T·C / (tasks · clusters) blocks).  ms_per_step is the MEASURED sample time."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cfg = synthetic.CONFIGS[args.config]
    from oracle import cofem as O
    n_t, n_c = {1: (4, 2), 2: (2, 4), 3: (1, 2), 4: (1, 1), 5: (1, 1), 6: (1, 2)}[args.config]
    data = synthetic.generate(cfg, range(n_t))
    sub = cfg.replace(C=n_c)
    data["cfg"] = sub
    data["pi"] = np.full(n_c, 1.0 / n_c)
    alpha = np.ones((n_c, cfg.D))
    times, steps = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        e = O.e_step(data, alpha, i, mode="cofem", T_global=cfg.T)
        alpha = O.m_step(e["q"], e["mu"], e["s"], alpha)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            steps.append(int(np.max(e["probe_steps"])))
    scale = (cfg.T * cfg.C) / (n_t * n_c)
    sample_ms = statistics.mean(times) * 1e3
    value = 1.0 / (sample_ms * 1e-3 * scale)
    bj = baseline_json()
    sample = (f"oracle (numpy fp64 cofem mode) EM iterations {args.warmup}..{args.warmup + args.steps - 1} on "
              f"{n_t} task(s) x {n_c} cluster(s) of {cfg.T} x {cfg.C} (EM and M-step over the sample; max CG "
              f"steps {max(steps)}); value = sample rate / {scale:.0f}")
    line = {"impl": "reference", "metric": bj["metric"], "value": value, "unit": "EM iters/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sample_ms, "ms_per_step_extrapolated": sample_ms * scale,
            "ms_per_step_note": "ms_per_step is the measured time of one sample EM iteration; "
                                "ms_per_step_extrapolated = 1000 / value (the configured workload)",
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name} (BASELINE.json configs[{cfg.cfg_id - 1}])", "T": cfg.T, "C": cfg.C,
                       "N": cfg.N, "D": cfg.D, "K": cfg.K, "cg_cap": cfg.cg_cap, "cg_tol": cfg.cg_tol,
                       "parallelism": "host cores"},
            "cpu_baseline": {"value": value, "unit": "EM iters/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "EM iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------------------
# CUDA arm
# --------------------------------------------------------------------------------------------
def ncu_traffic(cfg_name, engine="tensor"):
    """DRAM bytes (read + write) per CG step of the dominant kernel(s) — the persistent CG kernel
    (tensor engine) or the two operator SGEMM launches of a step (FP32 engine) — from the committed
    ncu --set full captures (profiles/ncu_summary.json), if any: the same unit as `achieved`."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            j = json.load(f)
        key = "traffic_bytes_per_cg_step_fp32" if engine == "fp32" else "traffic_bytes_per_cg_step"
        return j.get(key, {}).get(cfg_name)
    except Exception:
        return None


def cuda_arm(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            print("bench.py: --gpus N > 1 must be launched with torchrun (one rank per GPU)", file=sys.stderr)
            return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2310_00420_b200 import CoFEM, cmtcs

    cfg = synthetic.CONFIGS[args.config]
    engine = resolve_engine(args.engine, cfg)
    weak = world > 1 and args.scaling == "weak"
    t_total = cfg.T * world if weak else cfg.T
    if weak:   # rank r: global tasks [r·T, (r+1)·T) carrying the config's T tasks' Φ, y
        b, e = rank * cfg.T, (rank + 1) * cfg.T
        data = synthetic.generate(cfg)
    else:
        b, e = synthetic.shard(cfg.T, rank, world)
        data = synthetic.generate(cfg, range(b, e))
    pi = data["pi"]
    fourier = cfg.operator == "fourier"
    # the sensing operator's host copy: Φ (dense) or the sampled DFT rows Ω_t (partial Fourier)
    phi_h = torch.from_numpy(np.ascontiguousarray(data["rows"] if fourier else data["phi"])).pin_memory()
    y_h = torch.from_numpy(np.ascontiguousarray(data["y"])).pin_memory()
    del data
    phi = phi_h.to(dev)
    y = y_h.to(dev)
    uid = None
    if world > 1:
        obj = [cmtcs.cmtcs_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]

    def make(phi_d, y_d, alpha0=None, em_iter0=0, nccl_uid=None):
        if fourier:
            return CoFEM(None, y_d, fourier_rows=phi_d, D=cfg.D, T=t_total, C=cfg.C, K=cfg.K, beta=cfg.beta,
                         cg_max_iters=cfg.cg_cap, cg_rel_tol=cfg.cg_tol, probe_seed=cfg.probe_seed, pi=pi,
                         task_begin=b, nccl_uid=nccl_uid, rank=rank, world=world, alpha0=alpha0, em_iter0=em_iter0)
        return CoFEM(phi_d, y_d, T=t_total, C=cfg.C, K=cfg.K, beta=cfg.beta, cg_max_iters=cfg.cg_cap,
                     cg_rel_tol=cfg.cg_tol, probe_seed=cfg.probe_seed, pi=pi, task_begin=b,
                     shared_phi=cfg.shared_phi, nccl_uid=nccl_uid, rank=rank, world=world, alpha0=alpha0,
                     em_iter0=em_iter0, engine=engine)

    model = make(phi, y, nccl_uid=uid)
    stream = model.stream
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20), dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def allreduce(x: float, op) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    max_over_ranks = (lambda x: allreduce(x, dist.ReduceOp.MAX)) if world > 1 else (lambda x: x)
    min_over_ranks = (lambda x: allreduce(x, dist.ReduceOp.MIN)) if world > 1 else (lambda x: x)
    sum_over_ranks = (lambda x: allreduce(x, dist.ReduceOp.SUM)) if world > 1 else (lambda x: x)

    for _ in range(args.warmup):
        model.em_step(1)
    it0 = model.history[-1]["em_iter"] + 1 if model.history else 0
    alpha_snapshot = model.posterior()["alpha"].cpu().numpy() if model.history else np.ones((cfg.C, cfg.D))

    # ------------------------------ timed region (device-resident inputs) -------------------
    model.set_timing(True)
    model.get_timing(reset=True)
    launches0 = model.kernel_launches
    sampler = ClockSampler(local) if rank == 0 else None
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    infos = []
    barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.3)
    wall0 = time.perf_counter()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()                   # L2 flush between timed iterations (outside the events)
            evs[k][0].record(stream)
        infos.append(model.em_step(1))
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    barrier()
    clocks = sampler.stop() if sampler else None
    step_ms = [a.elapsed_time(bb) for a, bb in evs]
    rank_ms = sum(step_ms)
    total_ms = max_over_ranks(rank_ms)
    fastest_ms = min_over_ranks(rank_ms)
    tm = model.get_timing(reset=True)
    model.set_timing(False)
    launches = sum_over_ranks(model.kernel_launches - launches0)
    model.close()
    del model, flush
    torch.cuda.empty_cache()

    # algorithmic work: 4·N·D flop per active column per CG step
    col_iters = sum(i["probe_col_iters"] + i["mean_col_iters"] for i in infos)
    probe_iters = sum(i["probe_col_iters"] for i in infos)
    tile_iters = sum(i["tile_col_iters"] for i in infos)
    # dense: 4·N·D flop per active column per CG step (the two products with Φ_t);  partial Fourier:
    # two length-D complex FFTs, 5·D·log2(D) flop each (the standard radix-2 count), per column-step
    flop_per_col = (10.0 * cfg.D * math.log2(cfg.D)) if fourier else 4.0 * cfg.N * cfg.D
    flops_rank = flop_per_col * col_iters
    flops_all = sum_over_ranks(flops_rank)
    kern_ms = tm["cg_kernel_ms"]                 # the whole persistent CG kernel (CUDA events)
    op_ms = tm["op_ms"]                          # its operator phases only (device stamps)
    achieved = max_over_ranks(flops_rank / (kern_ms * 1e-3) / 1e12) if world == 1 else \
        sum_over_ranks(flops_rank / (kern_ms * 1e-3) / 1e12) / world
    achieved_op = flops_rank / (op_ms * 1e-3) / 1e12 if op_ms > 0 else 0.0
    peaks, peaks_kind = measured_peaks()
    peak_burst, peak_sust = tf32x3_peak_tflops(peaks)
    long_kernel = kern_ms / max(1, tm["cg_kernel_launches"]) > 1000.0
    peak = peak_sust if long_kernel else peak_burst
    alu = fourier or engine == "fp32"
    if alu:   # FP32 ALU bound (FFMA peak at the measured clock ceiling, B200_PROFILING.md unit counts)
        peak_burst = peak_sust = peak = fp32_peak_tflops(peaks.get("sm_max_mhz", SM_MAX_MHZ))
    # EM-step roofline (north_star): slower of Φ bytes at HBM bandwidth and FLOPs at peak, per CG step
    steps_total = sum(i["cg_iters"] for i in infos)
    phi_bytes = (4.0 * cfg.N if fourier else 4.0 * cfg.N * cfg.D) * (1 if cfg.shared_phi else (e - b)) * steps_total
    t_roof = max(flops_rank / (peak * 1e12), phi_bytes / (peaks["hbm_gbs"] * 1e9))
    em_roof_frac = max_over_ranks(t_roof) / (total_ms * 1e-3)

    # ------------------------------ end to end through the public API (host buffers) --------
    # the user's call sequence from pinned host memory: upload Φ, y; cmtcs_init (b = βΦᵀy, Φᵀ,
    # TMA maps) at the timed iterations' entry state; E EM iterations; posterior read back to host
    e2e = None
    if not args.no_e2e:
        ne = min(args.e2e_steps, args.steps) if args.e2e_steps > 0 else args.steps
        h2d = phi_h.numel() * phi_h.element_size() + y_h.numel() * 4 + cfg.C * cfg.D * 8
        d2h = ((e - b) * cfg.C + cfg.C * cfg.D + (e - b) * cfg.D + (e - b)) * 8
        barrier()
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream(dev)
        t0ev = torch.cuda.Event(enable_timing=True)
        t1ev = torch.cuda.Event(enable_timing=True)
        t0ev.record(cur)
        phi2 = torch.empty_like(phi_h, device=dev)
        y2 = torch.empty_like(y_h, device=dev)
        phi2.copy_(phi_h, non_blocking=True)
        y2.copy_(y_h, non_blocking=True)
        m2 = make(phi2, y2, alpha0=alpha_snapshot, em_iter0=it0, nccl_uid=uid)
        for _ in range(ne):
            m2.em_step(1)
        post = m2.posterior()
        host = {k: post[k].cpu() for k in ("q", "alpha", "recon", "assign")}
        t1ev.record(cur)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(t0ev.elapsed_time(t1ev))
        m2.close()
        del host, post, phi2, y2
        e2e = {"value": ne / (e2e_ms * 1e-3) * (world if weak else 1), "unit": "EM iters/s",
               "h2d_bytes_per_step": int(sum_over_ranks(h2d) / ne), "d2h_bytes_per_step": int(sum_over_ranks(d2h) / ne),
               "em_iters": ne, "em_iters_replayed": f"{it0}..{it0 + ne - 1}",
               "includes": "pinned-host -> device copy of Phi, y (and alpha0), cmtcs_init (b, Phi^T, tensor maps), "
                           "the EM iterations, posterior (q, alpha, recon, assign) device -> host"}

    if rank == 0:
        bj = baseline_json()
        value = args.steps / (total_ms * 1e-3) * (world if weak else 1)
        padded = tile_iters / max(probe_iters, 1)
        line = {
            "metric": bj["metric"], "value": value, "unit": "EM iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {
                "workload": f"{cfg.name} (BASELINE.json configs[{cfg.cfg_id - 1}])",
                "T": t_total, "T_per_rank": e - b, "C": cfg.C, "N": cfg.N, "D": cfg.D, "K": cfg.K,
                "cg_cap": cfg.cg_cap, "cg_tol": cfg.cg_tol, "em_iters_timed": f"{it0}..{it0 + args.steps - 1}",
                **({"value_definition": f"weak scaling: {world} ranks x {cfg.T} tasks; value = EM iterations/s "
                                        f"of the {t_total}-task job x {world} (config-sized EM iterations/s)"}
                   if weak else {}),
                "parallelism": f"task-sharded dp{world}" if world > 1 else "single GPU",
                "straggler_spread": (total_ms / fastest_ms) if world > 1 else 1.0,
                "engine": "partial-Fourier FFT" if fourier else engine,
                "precision": ("probe columns: fp32 vectors and fp32 FFT, fp64 dots/scalars; mean columns (fp64 FFT), "
                              "log-det, q, M-step fp64") if fourier else
                             ("probe columns: fp32 vectors, operator on the FP32 CUDA cores (FFMA, round-to-nearest, "
                              "two-level block sums), fp64 dots/scalars applied in fp64; mean columns, log-det, q, "
                              "M-step fp64") if engine == "fp32" else
                             ("probe columns: fp32 vectors, operator on tcgen05 tensor cores as 3xTF32 "
                              "(fp32-accurate), fp64 dots/scalars; mean columns, log-det, q, M-step fp64"),
                "l2": "flushed (zero-fill of 2xL2) between timed EM iterations",
                "cg_steps_per_em_iter": [i["cg_iters"] for i in infos],
                "active_col_iters_per_em_iter": [i["probe_col_iters"] + i["mean_col_iters"] for i in infos],
                "probe_tile_cols_multiplied_over_active": padded,
                "algorithmic_tflop_per_s_em": flops_all / (total_ms * 1e-3) / 1e12,
                "em_step_roofline_frac": em_roof_frac,
                "cg_kernel_share_of_step": kern_ms / max(rank_ms, 1e-9),
                # None: the FP32 engine runs two task halves as overlapping loops, phases are not separable
                "op_share_of_step": op_ms / max(rank_ms, 1e-9) if op_ms > 0 else None,
                "update_share_of_step": tm["update_ms"] / max(rank_ms, 1e-9) if op_ms > 0 else None,
                "wall_s_timed": wall,
            },
            "roofline": {"bound": "alu" if alu else "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(cfg.name, engine),
                         "traffic_unit": ("DRAM bytes per CG step (ncu --set full: k_simt_probe4<1> + k_simt_probe4<2>, "
                                          "one launch each)") if engine == "fp32" else
                                         "DRAM bytes per CG step (ncu --set full of k_cg_persistent / its CG steps)",
                         "kernel": ("k_cg_fourier (partial-Fourier CG: one CTA per column, FFT in shared memory; "
                                    "achieved = 10*D*log2(D) flop per active column per CG step / the kernels' "
                                    "duration)") if fourier else
                                   ("the FP32 engine's CG loop (k_simt_probe4<1>/<2> register-tiled SGEMMs for the "
                                    "probe columns, k_simt_mean<1/2> fp64 mean columns, k_simt_update); achieved = "
                                    "algorithmic fp32 flop 4*N*D per active column per CG step / the loop's duration "
                                    "(CUDA events on the launch stream around every E-step's CG loop); "
                                    "operator_phases_only: the same flops / the operator kernels' event time")
                                   if engine == "fp32" else
                                   ("k_cg_persistent (the whole CG loop of an E-step: operator on tcgen05 3xTF32 + fp64 "
                                    "mean columns on DMMA + CG update); achieved = algorithmic fp32 flop 4*N*D per "
                                    "active column per CG step / the kernel's duration (CUDA events on the launch "
                                    "stream around every launch in the timed region)"),
                         "peak_source": ("FFMA peak: 148 SMs x 128 FP32 lanes x 2 flop x sm_max_mhz "
                                         f"{peaks.get('sm_max_mhz', SM_MAX_MHZ)} (B200_PROFILING.md unit counts)")
                                        if alu else
                                        (f"{peaks_kind} MEASURED_PEAKS.json bf16 "
                                         f"{peaks['bf16_tflops_sustained' if long_kernel else 'bf16_tflops']} TF/s "
                                         f"({'sustained: kernel launches last > 1 s' if long_kernel else 'burst'}) "
                                         f"x (1.1/2.25 tf32/bf16 nominal) / 3 passes; burst {peak_burst:.1f}, "
                                         f"sustained {peak_sust:.1f}"),
                         "frac_burst_peak": achieved / peak_burst,
                         "operator_phases_only": None if op_ms <= 0 else
                                                 {"achieved": achieved_op, "frac": achieved_op / peak,
                                                  "timing": "CUDA events around the operator kernels of every CG step"
                                                  if engine == "fp32" else
                                                  "device %globaltimer stamps at the phase boundaries"},
                         "fp32_ffma_peak": fp32_peak_tflops(peaks.get("sm_max_mhz", SM_MAX_MHZ))},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        if e2e:
            line["e2e"] = e2e
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds, alpha_snapshot, it0)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    return cuda_arm(args)


if __name__ == "__main__":
    sys.exit(main())
