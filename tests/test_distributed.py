"""Multi-rank host logic on CPU (gloo, world size 2): task sharding, global-task probe streams and
the one all-reduce of the Eq. 4 sums give the single-process EM step exactly.

The GPU path does the same per rank (cmtcs_init with task_begin/task_end, ncclAllReduce of
[den (C·D), num (C), Σ log p(y_t)] inside cmtcs_em_step); only one GPU exists in this
environment, so the exchange algebra is exercised here with the oracle and torch.distributed/gloo.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic
from oracle import cofem as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synthetic.CONFIGS[1].replace(T=5, cluster_sizes=(3, 2))   # uneven shards: 3 + 2
    b, e = synthetic.shard(cfg.T, rank, world)
    data = synthetic.generate(cfg, range(b, e))
    alpha = np.random.default_rng(0).uniform(0.3, 3.0, (cfg.C, cfg.D))
    it = 3
    es = O.e_step(data, alpha, it, mode="cofem", T_global=cfg.T)      # probes keyed by global t
    num, den = O.m_step_sums(es["q"], es["mu"], es["s"])
    buf = torch.from_numpy(np.concatenate([den.ravel(), num, [np.sum(es["ll"])]]))
    dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    g = buf.numpy()
    C, D = cfg.C, cfg.D
    alpha_new = O.m_step_finish(g[C * D:C * D + C], g[:C * D].reshape(C, D), alpha)
    L = g[-1] / cfg.T
    # the id bytes the GPU path broadcasts from rank 0 travel intact through torch.distributed
    obj = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), alpha=alpha_new, L=L, mu=es["mu"], tasks=data["tasks"],
             uid_ok=obj[0] == bytes(range(128)))
    dist.destroy_process_group()


def test_two_rank_em_step_equals_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [np.load(tmp_path / f"r{i}.npz") for i in range(world)]
    cfg = synthetic.CONFIGS[1].replace(T=5, cluster_sizes=(3, 2))
    data = synthetic.generate(cfg)
    alpha = np.random.default_rng(0).uniform(0.3, 3.0, (cfg.C, cfg.D))
    es = O.e_step(data, alpha, 3, mode="cofem")
    want = O.m_step(es["q"], es["mu"], es["s"], alpha)
    for i in range(world):
        assert bool(r[i]["uid_ok"])
        np.testing.assert_allclose(r[i]["alpha"], want, rtol=1e-12)
        assert float(r[i]["L"]) == pytest.approx(es["L"], rel=1e-12)
    np.testing.assert_array_equal(np.concatenate([r[0]["tasks"], r[1]["tasks"]]), np.arange(cfg.T))
    np.testing.assert_allclose(np.concatenate([r[0]["mu"], r[1]["mu"]]), es["mu"], rtol=1e-12, atol=1e-14)
