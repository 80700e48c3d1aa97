"""Matrix Market / vector / permutation text I/O: the native parser's
verdicts equal the reference reader's on every golden case
(tests/golden/mmio_cases.json, made by make_mmio_golden.py from the
reference itself), write -> read round trips are bit-exact, and the native
fast path agrees with the exact slow path on large random files."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import ROOT

CASES = json.load(open(os.path.join(ROOT, "tests", "golden", "mmio_cases.json")))


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _verdict(fn):
    try:
        return {"ok": fn()}
    except Exception as e:  # noqa: BLE001
        return {"error": type(e).__name__, "message": str(e)}


def _readers():
    import paper_2407_17651_b200 as P
    return {
        "matrix": lambda p: (lambda r: [r[1], int(r[0].n), _digest(r[0].row, r[0].col, r[0].val)])(
            P.read_matrix(p)),
        "vector": lambda p: _digest(P.read_vector(p)),
        "permutation": lambda p: _digest(P.read_permutation(p).forward),
    }


@pytest.mark.parametrize("group,name", [(g, n) for g in CASES for n in CASES[g]])
def test_reader_matches_reference(group, name, tmp_path, lib_built):
    case = CASES[group][name]
    path = tmp_path / name
    with open(path, "w", encoding="ascii", newline="") as fh:
        fh.write(case["text"])
    want = {k: v for k, v in case.items() if k != "text"}
    got = _verdict(lambda: _readers()[group](str(path)))
    assert got == want


def _random_coo(n, nnz, seed):
    import paper_2407_17651_b200 as P
    rng = np.random.default_rng(seed)
    r = rng.integers(0, n, nnz)
    c = rng.integers(0, n, nnz)
    v = rng.standard_normal(nnz) * 10.0 ** rng.integers(-300, 300, nnz)
    v[::97] = 0.0
    v[1::101] = -0.0
    return P.coo_normalize(P.CooMatrix(n, r, c, v))


def test_general_round_trip_bit_exact(tmp_path, lib_built):
    import paper_2407_17651_b200 as P
    from paper_2407_17651_b200 import mmio
    m = _random_coo(5000, 200000, 1)
    p = tmp_path / "g.mtx"
    P.write_matrix(p, m)
    back, qual = P.read_matrix(p)
    assert qual == "general" and back.equals(m)
    slow, _ = mmio._exact_read_matrix(p)
    assert slow.equals(back)
    # signed zeros survive
    assert np.array_equal(np.signbit(back.val), np.signbit(m.val))


def test_skew_round_trip(tmp_path, lib_built):
    import paper_2407_17651_b200 as P
    from paper_2407_17651_b200 import generators as G
    g = G.stencil27(16, seed_val=3, alpha=0.0)
    m = P.SssMatrix(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    coo = P.sss_to_coo(m)
    p = tmp_path / "s.mtx"
    P.write_matrix(p, coo, "skew-symmetric")
    back, qual = P.read_matrix(p)
    assert qual == "skew-symmetric"
    assert P.coo_to_sss(back).equals(m)
    with pytest.raises(P.StructuralError, match="not strictly skew-symmetric"):
        P.write_matrix(p, P.CooMatrix(2, [1], [0], [1.0]), "skew-symmetric")
    with pytest.raises(ValueError, match="qualifier must be one of"):
        P.write_matrix(p, coo, "hermitian")


def test_vector_and_permutation_round_trip(tmp_path, lib_built):
    import paper_2407_17651_b200 as P
    x = np.random.default_rng(2).standard_normal(300000) * 1e-200
    x[7], x[8] = np.inf, -0.0
    P.write_vector(tmp_path / "x", x)
    y = P.read_vector(tmp_path / "x")
    assert np.array_equal(x, y) and np.signbit(y[8])
    fw = np.random.default_rng(3).permutation(100000)
    P.write_permutation(tmp_path / "p", P.Permutation(fw))
    assert np.array_equal(P.read_permutation(tmp_path / "p").forward, fw)
    with open(tmp_path / "p") as fh:
        assert fh.readline() == "100000\n" and fh.readline() == f"0 {fw[0]}\n"


def test_written_text_is_reference_format(tmp_path, lib_built):
    """Header, 1-based coordinates, "%.17g" values (mmio.py:183-187)."""
    import paper_2407_17651_b200 as P
    m = P.CooMatrix(3, [0, 2, 1], [0, 1, 2], [0.1, -1.0 / 3.0, 1e300])
    P.write_matrix(tmp_path / "m", m)
    lines = open(tmp_path / "m").read().splitlines()
    assert lines == ["%%MatrixMarket matrix coordinate real general", "3 3 3",
                     "1 1 %.17g" % 0.1, "2 3 %.17g" % 1e300, "3 2 %.17g" % (-1.0 / 3.0)]


def test_canonical_files_take_the_native_path(tmp_path, lib_built, monkeypatch):
    """Files in the writers' own format never fall back to the Python reader."""
    import paper_2407_17651_b200 as P
    from paper_2407_17651_b200 import mmio

    def boom(*a, **k):
        raise AssertionError("slow path used")
    monkeypatch.setattr(mmio, "_exact_read_matrix", boom)
    monkeypatch.setattr(mmio, "_exact_read_permutation", boom)
    m = _random_coo(300, 2000, 4)
    P.write_matrix(tmp_path / "m", m)
    assert P.read_matrix(tmp_path / "m")[0].equals(m)
    P.write_permutation(tmp_path / "p", P.Permutation(np.arange(50)[::-1]))
    assert P.read_permutation(tmp_path / "p").forward[0] == 49
