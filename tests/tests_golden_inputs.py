"""Input generators for the golden fixtures (same seeds as make_golden.py)."""

import numpy as np


def cfg3_small(n=120, split=20, rank=10):
    rng = np.random.default_rng(3)
    m = rng.standard_normal((n, n))
    u = rng.standard_normal((split, rank))
    v = rng.standard_normal((split, rank))
    m[:split, :split] = u @ v.T
    m[split:, split:] += float(n) * np.eye(n - split)
    return m


def _load_golden():
    from pathlib import Path

    return np.load(Path(__file__).resolve().parent / "golden" / "golden.npz")


GOLDEN = _load_golden()
