"""Shared fixtures: golden fixtures from the reference, the CPU oracle, helpers.

Markers: ``gpu`` -- needs a CUDA device (run with ``-m gpu`` on the B200 box);
everything else runs on CPU.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CORPUS_NAMES = ("tiny4", "one1", "zero3", "diag6", "tridiag5", "gen16", "gen64", "gen128shift",
                "gen257dense", "gen500")
PLAN_FIELDS = ("block_start", "row_owner", "safe_start", "conflict_idx", "conflict_ptr",
               "conflict_target", "apply_order", "apply_ptr", "halo_lo")
SPLIT_FIELDS = ("mid_ptr", "mid_col", "mid_val", "outer_row", "outer_col", "outer_val", "diag")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def lib_built():
    """Build libpars3.so once per session if it is missing (CPU-side tests
    need only its host functions)."""
    from paper_2407_17651_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import subprocess
        subprocess.run(["make", "-s", "-j8", "-C",
                        os.path.join(ROOT, "paper_2407_17651_b200", "csrc")], check=True)
    return _lib.load()


class GoldenCase:
    """One corpus member of tests/golden/corpus.npz (reference outputs)."""

    def __init__(self, z, name):
        self.name = name
        self._z = z
        self.n = int(z[f"{name}/n"][0])
        self.row_ptr = z[f"{name}/row_ptr"]
        self.col_ind = z[f"{name}/col_ind"]
        self.off_diags = z[f"{name}/off_diags"]
        self.diags = z[f"{name}/diags"]
        self.x = z[f"{name}/x"]
        self.y_serial = z[f"{name}/y_serial"]
        self.y_dense = z[f"{name}/y_dense"]
        self.rcm_forward = z[f"{name}/rcm_forward"]
        self.bandwidth = int(z[f"{name}/bandwidth"][0])
        self.betas = sorted({1, 4, max(1, self.bandwidth)})

    def ps(self):
        return [p for p in (1, 2, 3, 4, 8) if p <= self.n]

    def split(self, beta):
        return {f: self._z[f"{self.name}/b{beta}/{f}"] for f in SPLIT_FIELDS}

    def plan(self, beta, p):
        return {f: self._z[f"{self.name}/b{beta}/p{p}/{f}"] for f in PLAN_FIELDS}

    def y_pars3(self, beta, p):
        return self._z[f"{self.name}/b{beta}/p{p}/y_pars3"]

    def report(self, beta, p):
        return json.loads(bytes(self._z[f"{self.name}/b{beta}/p{p}/report"]).decode())


@pytest.fixture(scope="session")
def golden_corpus():
    z = dict(np.load(os.path.join(GOLDEN, "corpus.npz")))
    return {name: GoldenCase(z, name) for name in CORPUS_NAMES}


@pytest.fixture(scope="session")
def golden_c1():
    return dict(np.load(os.path.join(GOLDEN, "c1.npz")))


@pytest.fixture(scope="session")
def golden_hashes():
    with open(os.path.join(GOLDEN, "hashes.json")) as fh:
        return json.load(fh)


def sha(a) -> str:
    import hashlib
    a = np.ascontiguousarray(a)
    if a.dtype.kind in "iu":
        a = a.astype(np.int64)
    return hashlib.sha256(a.tobytes()).hexdigest()


def mixed_tol(ref, tol):
    """tol * max(1, ||ref||_inf) (reference tests/conftest.py:87-90)."""
    scale = max(1.0, float(np.max(np.abs(ref))) if np.size(ref) else 0.0)
    return tol * scale


def rel_err(y, ref):
    """||y - ref||_inf / max(1, ||ref||_inf) (cli.py:130-134, SPEC D14)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(y - ref)) / max(1.0, float(np.max(np.abs(ref)))))
