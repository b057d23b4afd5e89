"""CPU: the rest of the reference's public surface around the hot path --
matrix files (core.py:415-486), ProvisionalSet and the reference-signature
checkpoint functions (storage.py:166-411), the bench harness (bench.py) and
the CLI (cli.py) -- pinned to outputs of the reference itself
(tests/golden/make_golden.py).  No device needed: only host logic runs here;
compute paths are in tests/test_gpu_api.py."""

import importlib

import numpy as np
import pytest

from conftest import well_conditioned
from tests_golden_inputs import GOLDEN

import paper_2305_11103_b200 as bi
from paper_2305_11103_b200 import cli, storage
from paper_2305_11103_b200.errors import (
    BlockShapeMismatch,
    FormatError,
    InsufficientData,
    InvalidOrder,
    MissingProvisionalData,
)

B = importlib.import_module("paper_2305_11103_b200.bench")  # the package attribute is the bench() function


@pytest.mark.parametrize("kind", B.KINDS)
@pytest.mark.parametrize("order", [1, 5, 12])
def test_generate_equals_reference(kind, order):
    got = B.generate(order, seed=7, kind=kind)
    assert np.array_equal(got, GOLDEN[f"gen_{kind}_{order}"])


def test_generate_errors():
    with pytest.raises(InvalidOrder):
        B.generate(0)
    with pytest.raises(InvalidOrder):
        B.generate(4, kind="hilbert")


def _records():
    return [B.TimingRecord("a", o, 1, 1e-3 * (o / 8.0) ** 2.9 * (1.0 + 0.03 * ((o * 7) % 5)), 1e-13 * o)
            for o in (8, 16, 32, 64, 128)]


def test_fit_slope_and_csv_equal_reference():
    fit = B.fit_slope(_records(), 8, 128)
    ref = GOLDEN["bench_fit"]
    assert fit.n_points == int(ref[2])
    assert fit.exponent == pytest.approx(ref[0], rel=1e-12)
    assert fit.stderr == pytest.approx(ref[1], rel=1e-9)
    assert B.records_to_csv(_records()).encode() == GOLDEN["bench_csv"].tobytes()
    with pytest.raises(InsufficientData):
        B.fit_slope(_records(), 8, 32)


def test_bench_argument_errors():
    with pytest.raises(InvalidOrder):
        B.bench(["a"], [8], repeats=0)
    with pytest.raises(InvalidOrder):
        B.bench(["a"], [16, 8])
    with pytest.raises(InvalidOrder):
        B.bench(["lu"], [8])


def test_text_and_binary_matrix_files(tmp_path):
    m = well_conditioned(3, 5)
    bi.save_matrix(m, tmp_path / "m.txt")
    assert (tmp_path / "m.txt").read_bytes() == GOLDEN["text_file_3"].tobytes()
    assert np.array_equal(bi.load_matrix(tmp_path / "m.txt"), m)
    bi.save_matrix(m, tmp_path / "m.bin", binary=True)
    assert np.array_equal(bi.load_matrix(tmp_path / "m.bin"), m)  # magic sniffed
    (tmp_path / "bad1.txt").write_text("3\n1 2 3\n")
    (tmp_path / "bad2.txt").write_text("2 2\n1 2\n3\n")
    (tmp_path / "bad3.txt").write_text("1 2\n1 nan\n")
    (tmp_path / "bad4.txt").write_text("2 x\n1 2\n")
    for name in ("bad1.txt", "bad2.txt", "bad3.txt", "bad4.txt"):
        with pytest.raises(FormatError):
            bi.load_matrix(tmp_path / name)


def test_provisional_set_validation(tmp_path):
    scheme = bi.partition_from_sizes([3, 5, 2, 6])
    t = bi.ProvisionalSet(scheme, 1)
    assert t.n_quads == 2 and t.spans(1) == (2, 3, 4)
    t.store_l(0, np.zeros((5, 3)))
    t.store_r(1, np.zeros((2, 6)))
    t.store_s(3, np.ones((6, 6)))
    with pytest.raises(BlockShapeMismatch):
        t.store_l(0, np.zeros((3, 5)))
    with pytest.raises(MissingProvisionalData):
        t.r_block(0)
    assert [nm for nm, _ in t.entries()] == ["L_0", "R_1", "S_3"]
    with pytest.raises(BlockShapeMismatch):
        bi.ProvisionalSet(scheme, 3)
    f = bi.ProvisionalSet(scheme, 2, root=tmp_path / "t2")  # file-backed entries
    f.store_s(0, np.eye(8))
    assert (tmp_path / "t2" / "S_0.blk").exists()
    assert np.array_equal(f.s_block(0), np.eye(8))


def _golden_ckpt_files():
    return {k[len("ckpt4_file__"):].replace("__", "/"): GOLDEN[k].tobytes()
            for k in GOLDEN.files if k.startswith("ckpt4_file__")}


def test_reference_signature_checkpoint_roundtrip(tmp_path):
    """Load the reference-written directory through load_minv_store /
    load_tsets and write it back through storage.checkpoint_save with the
    reference's signature: every byte equal."""
    src = tmp_path / "src"
    for rel, data in _golden_ckpt_files().items():
        (src / rel).parent.mkdir(parents=True, exist_ok=True)
        (src / rel).write_bytes(data)
    scheme = bi.partition_from_sizes([8] * 4)
    meta = bi.checkpoint_load(src)
    minv = storage.load_minv_store(src, scheme)
    tsets = storage.load_tsets(src, scheme)
    m = well_conditioned(32, 61)
    assert storage.input_fingerprint(m, scheme) == meta["input_hash"]
    storage.checkpoint_matches(meta, scheme, meta["input_hash"])
    dst = tmp_path / "dst"
    bi.checkpoint_save(dst, scheme, minv, tsets, meta["stepid"], meta["input_hash"])
    files = _golden_ckpt_files()
    written = {str(p.relative_to(dst)): p.read_bytes() for p in dst.rglob("*") if p.is_file()}
    assert written == files
    store, fresh = storage.fresh_state(dst, scheme, file_backed=True)  # drops stale state (storage.py:391-411)
    assert not (dst / "meta.json").exists() and not list((dst / "tset").rglob("*.blk"))
    assert isinstance(store, storage.FileBlockStore)  # zeroed M_inv block files, as the reference writes them
    assert sorted(p.name for p in (dst / "minv").glob("*.blk")) == sorted(f"B_{i}_{j}.blk" for i in range(4)
                                                                          for j in range(4))
    assert np.count_nonzero(store.to_dense()) == 0 and set(fresh) == {1, 2}
    mem, _ = storage.fresh_state(dst, scheme, file_backed=False)
    assert np.count_nonzero(mem.data) == 0


def test_cli_parser_and_host_commands(tmp_path, capsys):
    assert cli.order_list("8:32:8") == [8, 16, 24, 32] and cli.int_list("4,,8") == [4, 8]
    assert cli.main(["partition", "12"]) == 0
    out = capsys.readouterr().out
    assert "order 12: N_k = 4 diagonal blocks, 7 steps" in out and "sizes 3 3 3 3" in out
    assert cli.main(["partition", "0", "--sizes", "5,7"]) == 0
    assert "N_k = 2" in capsys.readouterr().out
    path = tmp_path / "g.bin"
    assert cli.main(["gen", "--order", "12", "--seed", "7", "--kind", "block-diagonal", "--out", str(path),
                     "--binary"]) == 0
    assert np.array_equal(bi.load_matrix(path), GOLDEN["gen_block-diagonal_12"])
    # I/O and format errors map to exit code 3 before any device work
    assert cli.main(["invert", "--in", str(tmp_path / "missing.txt")]) == cli.EXIT_IO
    (tmp_path / "bad.txt").write_text("2 2\n1 2\n")
    assert cli.main(["invert", "--in", str(tmp_path / "bad.txt")]) == cli.EXIT_IO
    assert cli.main(["partition", "1"]) == cli.EXIT_IO  # InvalidOrder
    with pytest.raises(SystemExit):
        cli.main(["invert", "--in", "x", "--method", "lu"])


def test_file_block_store_roundtrip(tmp_path):
    """FileBlockStore (storage.py:73-125): one BMAT file per block, region
    reads/writes across block boundaries, BlockMatrix.from_dense(directory=)."""
    scheme = bi.partition_from_sizes([3, 5, 2, 6])
    g = np.random.default_rng(3)
    m = g.standard_normal((16, 16))
    bm = storage.BlockMatrix.from_dense(m, scheme, directory=tmp_path / "blocks")
    assert isinstance(bm.store, storage.FileBlockStore) and bm.store.file_backed
    assert sorted(p.name for p in (tmp_path / "blocks").glob("*.blk")) == sorted(
        f"B_{i}_{j}.blk" for i in range(4) for j in range(4))
    assert np.array_equal(bm.to_dense(), m)
    off = scheme.offsets
    assert np.array_equal(bm.store.region(1, 3, 0, 2), m[off[1]:off[3], off[0]:off[2]])
    vals = g.standard_normal((off[3] - off[1], off[4] - off[2]))
    bm.store.set_region(1, 3, 2, 4, vals)
    m2 = m.copy()
    m2[off[1]:off[3], off[2]:off[4]] = vals
    assert np.array_equal(bm.to_dense(), m2)
    assert np.array_equal(storage.FileBlockStore(scheme, tmp_path / "blocks").to_dense(), m2)  # reopened
