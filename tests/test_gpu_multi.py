"""The one-process-per-GPU driver of the column-sharded level scheduler
(distributed.sharded_engine -> NativeShardDist), launched the way
``bench.py --gpus N`` launches it: torchrun, one rank per GPU.

* two NCCL ranks on two GPUs, both transports (torch.distributed all-gathers
  and NCCL inside the library, bi_engine_run_nccl): runs whenever at least
  two GPUs are visible, skipped otherwise (the round's GPU boxes have one);
* the same worker with two and four ranks sharing the visible GPU over gloo:
  runs on every GPU box, so the driver, the group construction, the
  pack / all-gather / unpack exchanges, gather-to-rank-0 and the collective
  singular-leaf report are exercised even without a second GPU.

The worker (tests/_shard_worker.py) compares rank 0's gathered inverse
bitwise with the single-GPU engine and within 1e-12 n with the CPU oracle.
"""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
WORKER = ROOT / "tests" / "_shard_worker.py"


def _torchrun(nproc: int, env_extra: dict) -> subprocess.CompletedProcess:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env.update(env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(WORKER)]
    return subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)


def _gpus() -> int:
    import torch

    return torch.cuda.device_count()


@pytest.mark.parametrize("nproc", [2, 4])
def test_sharded_driver_ranks_sharing_one_gpu_gloo(nproc):
    r = _torchrun(nproc, {"BI_TEST_SHARE_GPU": "1"})
    assert r.returncode == 0 and "SHARD_WORKER_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])


@pytest.mark.parametrize("transport", ["torch", "lib"])
def test_sharded_driver_nccl_one_rank_per_gpu(transport):
    n = _gpus()
    if n < 2:
        pytest.skip(f"needs at least 2 GPUs (NCCL refuses two ranks on one device); {n} visible")
    nproc = 4 if n >= 4 else 2
    extra = {"BI_SHARD_TRANSPORT": "lib"} if transport == "lib" else {}
    r = _torchrun(nproc, extra)
    assert r.returncode == 0 and "SHARD_WORKER_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])
