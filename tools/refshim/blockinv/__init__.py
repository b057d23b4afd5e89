"""Import shim: the reference package name ``blockinv`` resolved to this
framework, so the reference's own test suite (/root/reference/pkg/tests,
``from blockinv.engine import run_inversion`` ...) runs against the B200
implementation unchanged.  Used only by tools/reference_suite.py."""

import importlib
import sys

_PKG = "paper_2305_11103_b200"
for _name in ("core", "engine", "schur", "recursive", "partition", "storage", "errors", "cli", "bench"):
    _mod = importlib.import_module(f"{_PKG}.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

from paper_2305_11103_b200 import *  # noqa: E402,F401,F403
