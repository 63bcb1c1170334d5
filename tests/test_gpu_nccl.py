"""The library's NCCL path (ncclCommInitRank + the per-EM-iteration ncclAllReduce of the Eq. 4
sums, csrc/cmtcs_api.cu) on >= 2 GPUs: a sharded run equals a single-context run.  Skipped on a
1-GPU box (the shard algebra itself is covered there by test_task_shards_match_whole, which
compares each shard context's pre-all-reduce sums, cmtcs_estep_sums, with the whole problem's)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_nccl_allreduce_sharded_run_matches_single_context():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(HERE, "nccl_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0
