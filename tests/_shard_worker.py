"""One rank of a torchrun-launched run of the column-sharded level scheduler
(SURVEY 8e), the path ``bench.py --gpus N`` takes: one process per GPU,
``distributed.sharded_engine`` (NativeShardDist over shard.NativeShard), the
global-level exchanges as all-gathers inside the rank groups, the inverse
gathered to rank 0.  Started by tests/test_gpu_multi.py.

    BI_TEST_SHARE_GPU=1   ranks share the visible GPUs and exchange over gloo
                          (NCCL refuses two ranks on one device): the worker's
                          own check on a 1-GPU box
    BI_SHARD_TRANSPORT=lib  the exchanges as NCCL calls inside the library
                          (bi_engine_run_nccl) instead of torch.distributed

Rank 0 compares the gathered inverse with the single-GPU engine (bitwise: K
is never split, reference tests/test_acceptance.py:146-156) and with the CPU
oracle engine, then prints SHARD_WORKER_OK.
"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main() -> None:
    import torch
    import torch.distributed as dist

    share = os.environ.get("BI_TEST_SHARE_GPU") == "1"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if share:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import oracle
    import paper_2305_11103_b200 as bi
    from conftest import well_conditioned
    from paper_2305_11103_b200.distributed import sharded_engine

    cases = [([64] * 8, None), ([40, 72, 56, 24, 88, 48, 64, 32], None), ([32] * 16, 11)]
    for sizes, stop in cases:
        if len(sizes) % world:
            continue
        n = sum(sizes)
        m = well_conditioned(n, 700 + n)
        eng = sharded_engine(sizes)
        eng.load(m)
        eng.run(1, stop)
        eng.check()
        full = eng.gather(0)
        assert eng.launches() > 0
        if rank == 0:
            single = bi.run_inversion(m, sizes=sizes, stop_after_step=stop).to_dense()
            assert np.array_equal(full, single), ("sharded != single engine", sizes, stop)
            if stop is None:
                ref = oracle.run_inversion(m, sizes=sizes, leaf_inverter=oracle.gauss_jordan)
                assert np.max(np.abs(full - ref)) <= 1e-12 * n
        else:
            assert full is None
        dist.barrier()

    # a singular leaf: every rank raises the earliest SingularBlock(step, quad)
    sizes = [16] * 8
    n = sum(sizes)
    m = well_conditioned(n, 5)
    m[80:96, 80:96] = 0.0
    eng = sharded_engine(sizes)
    eng.load(m)
    eng.run()
    try:
        eng.check()
    except bi.SingularBlock as exc:
        assert (exc.step, exc.quad) == (1, 5), (exc.step, exc.quad)
    else:
        raise AssertionError("singular leaf not reported")
    dist.barrier()
    if rank == 0:
        print("SHARD_WORKER_OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
