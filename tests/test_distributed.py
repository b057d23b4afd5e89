"""Multi-process tests of the column-sharded level scheduler.

CPU (gloo, world sizes 2 and 4): the schedule, ownership and collectives of
paper_2305_11103_b200.distributed run with a torch-CPU compute backend defined
here (test infrastructure), checked against the oracle engine.
GPU: two processes share the one B200 (gloo collectives, B200 kernels) and
must reproduce the single-device engine bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import well_conditioned


class TorchCPUBackend:
    """float64 torch-CPU primitives with the oracle's pivoted GJ leaf."""

    def empty(self, rows, cols):
        return torch.empty((rows, cols), dtype=torch.float64)

    def gemm(self, a, b, d, c=None, negate=False):
        prod = a @ b
        res = (c.clone() if c is not None else torch.zeros_like(d)) + (-prod if negate else prod)
        d.copy_(res)

    def inverse(self, blocks, outs):
        info = np.zeros(blocks.shape[0], dtype=np.int32)
        for i in range(blocks.shape[0]):
            try:
                outs[i].copy_(torch.from_numpy(oracle.gauss_jordan(blocks[i].numpy())))
            except oracle.OracleSingularMatrix:
                info[i] = 1
        return info


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, sizes, seed, device, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_11103_b200.distributed import run_inversion_sharded

        n = sum(sizes)
        m = well_conditioned(n, seed)
        backend = TorchCPUBackend() if not device else None
        if device:
            torch.cuda.set_device(0)
        inv = run_inversion_sharded(m, sizes, backend=backend)
        q.put((rank, inv))
    except Exception as exc:  # surface worker failures in the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def _run(world, sizes, seed, device=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sizes, seed, device, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, v = q.get(timeout=600)
        out[r] = v
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        assert not isinstance(v, str), f"rank {r}: {v}"
    return out


@pytest.mark.parametrize("world,sizes", [(2, [6] * 4), (2, [5, 7, 6, 4, 8, 3, 5, 6]), (2, [3, 9, 2, 4]),
                                         (4, [8] * 8), (4, [2, 7, 5, 3, 6, 4, 9, 1])])
def test_sharded_schedule_cpu_gloo(world, sizes):
    n = sum(sizes)
    seed = 900 + n
    out = _run(world, sizes, seed)
    ref = oracle.run_inversion(well_conditioned(n, seed), sizes=sizes, leaf_inverter=oracle.gauss_jordan)
    assert np.max(np.abs(out[0] - ref)) <= 1e-12 * n
    assert all(out[r] is None for r in range(1, world))  # gathered on the root only


@pytest.mark.gpu
def test_sharded_two_ranks_one_gpu_bitwise():
    import paper_2305_11103_b200 as bi

    sizes = [64] * 8
    n = sum(sizes)
    seed = 77
    out = _run(2, sizes, seed, device=True)
    single = bi.run_inversion(well_conditioned(n, seed), sizes=sizes).to_dense()
    assert np.array_equal(out[0], single)
    assert out[1] is None


# --- one process, one thread per GPU (run_inversion(workers=P), local_group.py) ---

@pytest.mark.parametrize("gpus,sizes", [(2, [6] * 4), (2, [5, 7, 6, 4, 8, 3, 5, 6]), (4, [8] * 8),
                                        (4, [2, 7, 5, 3, 6, 4, 9, 1])])
def test_local_threads_schedule_cpu(gpus, sizes):
    from paper_2305_11103_b200.distributed import run_inversion_local

    n = sum(sizes)
    m = well_conditioned(n, 950 + n)
    out = run_inversion_local(m, sizes, gpus, backend_factory=TorchCPUBackend, devices=[None] * gpus)
    ref = oracle.run_inversion(m, sizes=sizes, leaf_inverter=oracle.gauss_jordan)
    assert np.max(np.abs(out - ref)) <= 1e-12 * n


class FusedCPUBackend(TorchCPUBackend):
    """TorchCPUBackend plus the K1P entry (segments concatenated on the host):
    drives the fused-exchange schedule (share -> in-place segment reads ->
    release) on CPU threads."""

    kseg_align = 1
    calls = 0

    def gemm_kseg(self, segs, b, d, c=None, negate=False):
        type(self).calls += 1
        self.gemm(torch.cat(list(segs), dim=1), b, d, c=c, negate=negate)


@pytest.mark.parametrize("gpus,sizes,align", [(2, [6] * 4, 1), (4, [8] * 8, 1), (4, [2, 7, 5, 3, 6, 4, 9, 1], 1),
                                              (4, [4, 4, 5, 3, 6, 2, 4, 4], 8)])
def test_local_threads_fused_exchange_cpu(monkeypatch, gpus, sizes, align):
    """Global levels read the peers' slabs as K segments (no gathered copy);
    same inverse as the oracle engine.  With align=8 the ragged group whose
    first owner is 8 wide fuses and the rest falls back to the all-gather."""
    from paper_2305_11103_b200.distributed import run_inversion_local

    monkeypatch.setenv("BI_FUSED_GATHER", "1")

    class B(FusedCPUBackend):
        kseg_align = align
        calls = 0

    n = sum(sizes)
    m = well_conditioned(n, 970 + n)
    out = run_inversion_local(m, sizes, gpus, backend_factory=B, devices=[None] * gpus)
    ref = oracle.run_inversion(m, sizes=sizes, leaf_inverter=oracle.gauss_jordan)
    assert np.max(np.abs(out - ref)) <= 1e-12 * n
    assert B.calls > 0


def test_local_threads_failure_does_not_hang():
    from paper_2305_11103_b200.distributed import run_inversion_local

    class Failing(TorchCPUBackend):
        def inverse(self, blocks, outs):
            raise RuntimeError("leaf failure on purpose")

    with pytest.raises(RuntimeError, match="on purpose"):
        run_inversion_local(well_conditioned(24, 3), [6] * 4, 2, backend_factory=Failing, devices=[None] * 2)


def test_workers_to_gpu_count(monkeypatch):
    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.engine import gpus_for_workers

    t = _lib.torch()
    monkeypatch.setattr(t.cuda, "is_available", lambda: True)
    monkeypatch.setattr(t.cuda, "device_count", lambda: 8)
    assert gpus_for_workers(None, 8) == 1 and gpus_for_workers(1, 8) == 1
    assert gpus_for_workers(8, 8) == 8 and gpus_for_workers(8, 64) == 8
    assert gpus_for_workers(6, 8) == 4 and gpus_for_workers(16, 8) == 8
    assert gpus_for_workers(8, 4) == 4 and gpus_for_workers(8, 2) == 2
    assert gpus_for_workers(4, 1) == 1  # one diagonal block: nothing to shard
    monkeypatch.setattr(t.cuda, "device_count", lambda: 2)
    assert gpus_for_workers(8, 8) == 2


@pytest.mark.gpu
def test_local_threads_two_on_one_gpu_bitwise():
    """Two threads sharing the B200 run the sharded schedule with peer-copy
    exchanges: bitwise equal to the single-device engine."""
    import paper_2305_11103_b200 as bi
    from paper_2305_11103_b200.distributed import run_inversion_local

    sizes = [64] * 8
    m = well_conditioned(512, 78)
    out = run_inversion_local(m, sizes, 2, devices=[0, 0])
    single = bi.run_inversion(m, sizes=sizes).to_dense()
    assert np.array_equal(out, single)


@pytest.mark.gpu
@pytest.mark.parametrize("gpus,sizes,fused", [(2, [64] * 8, "1"), (2, [64] * 8, "0"), (4, [128] * 8, "1"),
                                              (4, [40, 24, 64, 56, 72, 8, 48, 32], "1")])
def test_local_threads_fused_gather_bitwise(monkeypatch, gpus, sizes, fused):
    """K1P inside the thread-per-GPU schedule (threads sharing the B200, each
    reading the others' slabs through their device pointers): bitwise equal
    to the single-device engine, fused (BI_FUSED_GATHER=1, opt-in) or with
    the gathered copies (0, default); the fused run really takes K1P."""
    import paper_2305_11103_b200 as bi
    from paper_2305_11103_b200 import distributed
    from paper_2305_11103_b200.distributed import run_inversion_local

    monkeypatch.setenv("BI_FUSED_GATHER", fused)
    calls = []
    orig = distributed.DeviceBackend.gemm_kseg

    def counting(self, *a, **k):
        calls.append(1)
        return orig(self, *a, **k)

    monkeypatch.setattr(distributed.DeviceBackend, "gemm_kseg", counting)
    n = sum(sizes)
    m = well_conditioned(n, 79 + gpus)
    out = run_inversion_local(m, sizes, gpus, devices=[0] * gpus)
    single = bi.run_inversion(m, sizes=sizes).to_dense()
    assert np.array_equal(out, single)
    assert (len(calls) > 0) == (fused == "1")


@pytest.mark.parametrize("stop,expect", [(0, 1), (-3, 1), (3, 3), (7 + 5, 7)])
def test_local_threads_stop_after_step_clamped(stop, expect):
    """stop_after_step outside 1..N_s is clamped like the reference and the
    single-device engine (at least one step, at most N_s): ADVICE r01."""
    from paper_2305_11103_b200.distributed import run_inversion_local

    sizes = [6] * 4  # N_s = 7
    n = sum(sizes)
    m = well_conditioned(n, 321)
    out = run_inversion_local(m, sizes, 2, stop_after_step=stop, backend_factory=TorchCPUBackend,
                              devices=[None] * 2)
    ref = oracle.run_inversion(m, sizes=sizes, leaf_inverter=oracle.gauss_jordan, stop_after_step=expect)
    assert np.max(np.abs(out - ref)) <= 1e-12 * n
