"""Small launches of every race-prone kernel, for compute-sanitizer
(racecheck / memcheck / synccheck), one tool per gpurun call:

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

cases: k1_tma (K1 TMA refill ring, 2 CTAs/SM tiles), k1_cp (cp.async feeder,
unaligned view), k3_panel (8 x 256 and 4 x 512 leaves: register panels, K1
updates, gathers), k3_cluster (1 x 1000: cluster-resident outer panel with
the DSMEM argmax), kseg (K1P, 3 segments), kseg_mc (K1P with a 2-CTA TMA
multicast cluster, BI_KSEG_CLUSTER=2), engine (a 16 x 24-block run_inversion:
every engine op), shard (2 column-sharded ranks on one GPU, bi_shard_group_run).
Each case checks its result so a silent corruption also fails.
"""

import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main(cases):
    import torch

    import oracle
    import paper_2305_11103_b200 as bi
    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import device_gemm, device_gemm_kseg, device_inverse

    g = np.random.default_rng(1)
    dev = lambda a: _lib.to_device(a)  # noqa: E731
    for case in cases:
        if case in ("k1_tma", "k1_cp"):
            m, k, n = (256, 256, 320) if case == "k1_tma" else (130, 77, 201)
            a, b, c = g.standard_normal((m, k)), g.standard_normal((k, n)), g.standard_normal((m, n))
            da, db, dc = dev(a), dev(b), dev(c)
            if case == "k1_cp":
                da = dev(np.pad(a, ((0, 0), (1, 0))))[:, 1:]  # 8-byte aligned view: cp.async feeder
            dd = _lib.empty_matrix(m, n)
            device_gemm(da, db, dd, c=dc, negate=True)
            assert np.allclose(dd.cpu().numpy(), c - a @ b, atol=1e-12)
        elif case in ("k3_panel", "k3_cluster"):
            for cnt, nn in ((8, 256), (4, 512)) if case == "k3_panel" else ((1, 1000),):
                x = g.standard_normal((cnt, nn, nn)) + nn * np.eye(nn)
                dx = dev(x)
                do = _lib.empty_matrix(nn, nn, batch=cnt)
                info = device_inverse(dx, do)
                assert not np.any(np.asarray(info.cpu() if hasattr(info, "cpu") else info))
                for i in range(cnt):
                    assert oracle.rel_frob(do[i].cpu().numpy(), np.linalg.inv(x[i])) <= 1e-12
        elif case in ("kseg", "kseg_mc"):
            if case == "kseg_mc":
                os.environ["BI_KSEG_CLUSTER"] = "2"
            m, n = 256, 192
            ws = [64, 128, 48]
            segs = [g.standard_normal((m, w)) for w in ws]
            b = g.standard_normal((sum(ws), n))
            dd = _lib.empty_matrix(m, n)
            device_gemm_kseg([dev(s) for s in segs], dev(b), dd)
            assert np.allclose(dd.cpu().numpy(), np.hstack(segs) @ b, atol=1e-12)
        elif case == "engine":
            sizes = [24] * 16
            nn = sum(sizes)
            x = g.uniform(-1, 1, (nn, nn)) + 2 * nn * np.eye(nn)
            inv = bi.run_inversion(x, sizes=sizes).to_dense()
            assert oracle.rel_frob(inv, np.linalg.inv(x)) <= 1e-12
        elif case == "shard":
            from paper_2305_11103_b200.shard import run_inversion_group

            sizes = [24] * 8
            nn = sum(sizes)
            x = g.uniform(-1, 1, (nn, nn)) + 2 * nn * np.eye(nn)
            got = run_inversion_group(x, sizes, 2, devices=[0, 0])
            assert np.array_equal(got, bi.run_inversion(x, sizes=sizes).to_dense())
        else:
            raise SystemExit(f"unknown case {case}")
        torch.cuda.synchronize()
        print(f"case {case}: ok", flush=True)


if __name__ == "__main__" and not os.environ.get("BI_STRESS"):
    main(sys.argv[1:] or ["k1_tma", "k1_cp", "k3_panel", "k3_cluster", "kseg", "kseg_mc", "engine", "shard"])


def stress(reps: int = 200) -> None:
    """compute-sanitizer is closed on this pool, so races are hunted as
    nondeterminism: every race-prone kernel is re-run ``reps`` times on the
    same inputs (with other work interleaved to perturb timing) and must be
    bitwise identical every time."""
    import torch

    import paper_2305_11103_b200 as bi
    from paper_2305_11103_b200 import _lib
    from paper_2305_11103_b200.core import device_gemm, device_gemm_kseg, device_inverse

    g = np.random.default_rng(2)
    dev = lambda a: _lib.to_device(a)  # noqa: E731
    noise = torch.empty((1 << 26,), dtype=torch.float64, device="cuda")
    results = {}

    def check(name, fn):
        ref = fn()
        bad = 0
        for i in range(reps):
            if i % 3 == 0:
                noise.mul_(1.0000001)  # perturb timing / L2 state between replays
            if not torch.equal(fn(), ref):
                bad += 1
        results[name] = bad
        print(f"stress {name}: {reps} replays, {bad} differ", flush=True)

    a, b, c = (dev(g.standard_normal(s)) for s in ((1024, 768), (768, 1280), (1024, 1280)))
    d = _lib.empty_matrix(1024, 1280)
    check("k1_tma_refill", lambda: (device_gemm(a, b, d, c=c), d.clone())[1])
    af, bf = dev(g.standard_normal((2560, 1024))), dev(g.standard_normal((1024, 4096)))
    df = _lib.empty_matrix(2560, 4096)
    check("k1_fat_4warp", lambda: (device_gemm(af, bf, df), df.clone())[1])  # K >= 1024, 1280 tiles
    x64 = dev(g.standard_normal((64, 256, 256)) / 16 + 4 * np.eye(256))
    o64 = _lib.empty_matrix(256, 256, batch=64)
    check("k3_64x256", lambda: (device_inverse(x64, o64), o64.clone())[1])
    segs = [dev(g.standard_normal((512, w))) for w in (128, 256, 64)]
    bb = dev(g.standard_normal((448, 384)))
    dk = _lib.empty_matrix(512, 384)
    os.environ["BI_KSEG_CLUSTER"] = "2"
    check("k1p_multicast", lambda: (device_gemm_kseg(segs, bb, dk), dk.clone())[1])
    x = dev(g.standard_normal((8, 512, 512)) + 512 * np.eye(512))
    o = _lib.empty_matrix(512, 512, batch=8)
    check("k3_panels_8x512", lambda: (device_inverse(x, o), o.clone())[1])
    x1 = dev(g.standard_normal((1, 1500, 1500)) + 1500 * np.eye(1500))
    o1 = _lib.empty_matrix(1500, 1500, batch=1)
    check("k3_cluster_1x1500", lambda: (device_inverse(x1, o1), o1.clone())[1])
    sizes = [64] * 16
    m = g.uniform(-1, 1, (1024, 1024)) + 2048 * np.eye(1024)
    eng = bi.DeviceEngine(sizes)
    eng.load(m)
    check("engine_graph", lambda: (eng.run(), eng.Minv.clone())[1])
    assert not any(results.values()), results


if __name__ == "__main__" and os.environ.get("BI_STRESS"):
    stress(int(os.environ["BI_STRESS"]))
