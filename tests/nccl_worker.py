"""Worker of tests/test_gpu_nccl.py (launched by torchrun, one rank per GPU): runs config 1 sharded
over the ranks through libcmtcs with its NCCL all-reduce of the Eq. 4 sums (the
north_star's one collective), and on rank 0 compares α and the log-likelihood with a single-context
run of the whole problem on the same GPU."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synthetic  # noqa: E402
from gpu_common import make_gpu, to_np  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    from paper_2310_00420_b200 import CoFEM, cmtcs
    cfg = synthetic.CONFIGS[1]
    b, e = synthetic.shard(cfg.T, rank, world)
    part = synthetic.generate(cfg, range(b, e))
    obj = [cmtcs.cmtcs_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    m = CoFEM(torch.from_numpy(part["phi"]).cuda(), torch.from_numpy(part["y"]).cuda(), T=cfg.T, C=cfg.C,
              K=cfg.K, beta=cfg.beta, cg_max_iters=256, cg_rel_tol=cfg.cg_tol, probe_seed=cfg.probe_seed,
              task_begin=b, nccl_uid=obj[0], rank=rank, world=world)
    infos = [m.em_step(1) for _ in range(3)]
    alpha = to_np(m.posterior())["alpha"]
    m.close()
    ok = True
    if rank == 0:
        data = synthetic.generate(cfg)
        w = make_gpu(data, cap=256)
        winfos = [w.em_step(1) for _ in range(3)]
        wa = to_np(w.posterior())["alpha"]
        w.close()
        da = float(np.max(np.abs(alpha - wa) / np.abs(wa)))
        dl = max(abs(a["loglik"] - b_["loglik"]) for a, b_ in zip(infos, winfos))
        print(f"NCCL world {world}: max rel |d alpha| {da:.3e}, max |d loglik| {dl:.3e}", flush=True)
        ok = da <= 1e-9 and dl <= 1e-8   # summation order of the two partial sums only
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(t, 0)
    dist.destroy_process_group()
    sys.exit(0 if int(t.item()) == 1 else 1)


if __name__ == "__main__":
    main()
