"""Instrumented protocol models and the reference's smaller public pieces,
pinned to the reference's own outputs (tests/golden/instrument_cases.json,
made by make_instrument_golden.py): traces of spmv_pars3_instrumented
(messages, stage log, tallies, bit-exact y), spmv_serial_instrumented,
generate_band_skew, CsrMatrix / coo_to_csr."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from conftest import CORPUS_NAMES, ROOT

CASES = json.load(open(os.path.join(ROOT, "tests", "golden", "instrument_cases.json")))


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _corpus(name):
    z = np.load(os.path.join(ROOT, "tests", "golden", "corpus.npz"))
    n = int(z[f"{name}/n"][0])
    m = P.SssMatrix(n, z[f"{name}/row_ptr"], z[f"{name}/col_ind"], z[f"{name}/off_diags"],
                    z[f"{name}/diags"])
    return m, z[f"{name}/x"]


@pytest.mark.parametrize("name", CORPUS_NAMES)
def test_serial_instrumented_matches_reference(name):
    m, x = _corpus(name)
    y, ops = P.spmv_serial_instrumented(m, x)
    want = CASES["serial"][name]
    assert _digest(y) == want["y"]
    assert [ops.element_reads, ops.multiply_adds] == want["ops"]


@pytest.mark.parametrize("key", sorted(CASES["pars3"]))
def test_pars3_trace_matches_reference(key, lib_built):
    name, b, p = key.split("/")
    m, x = _corpus(name)
    s = P.split_bands(m, int(b[1:]))
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, int(p[1:])))
    t = P.spmv_pars3_instrumented(s, plan, x)
    want = CASES["pars3"][key]
    assert _digest(t.y) == want["y"]
    assert [[mm.target_worker, mm.target_row, mm.value.hex(), mm.source_worker, mm.source_row,
             mm.source_col, mm.slot] for mm in t.messages] == want["messages"]
    assert [list(e) for e in t.stage_log] == want["stage_log"]
    assert [[c.worker_id, c.row_start, c.row_end, c.halo_lo, c.element_reads, c.multiply_adds,
             c.stages, len(c.outbox)] for c in t.contexts] == want["contexts"]
    assert [t.coordinator_reads, t.coordinator_multiply_adds, t.outer_count] == want["coordinator"]
    assert [t.total_ops().element_reads, t.total_ops().multiply_adds] == want["total"]
    assert t.message_count == len(want["messages"])


def test_trace_y_equals_oracle_pars3(oracle, lib_built):
    """Bit-identical to the pinned C restatement of _pars3 on a larger case."""
    from paper_2407_17651_b200 import generators as G
    g = G.random_band(3000, 100, 6, 0.02, seed_struct=1, seed_perm=2, seed_val=3)
    m = P.SssMatrix(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    s = P.split_bands(m, 20)
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 4))
    x = G.make_x(m.n, 4)
    t = P.spmv_pars3_instrumented(s, plan, x)
    split = {"n": s.n, "beta": s.beta, "mid_ptr": s.mid_ptr, "mid_col": s.mid_col.astype(np.int64),
             "mid_val": s.mid_val, "diag": s.diag, "outer_row": s.outer_row.astype(np.int64),
             "outer_col": s.outer_col.astype(np.int64), "outer_val": s.outer_val}
    po = oracle.classify_conflicts(split, oracle.partition_rows(s.n, 4))
    assert np.array_equal(t.y, oracle.spmv_pars3(split, po, x))
    y2, _ = P.spmv_serial_instrumented(m, x)
    assert np.array_equal(y2, oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x))


def test_worker_context_guards():
    ctx = P.WorkerContext(1, 4, 8, 2, np.zeros(4), local_x=np.arange(4.0), local_y=np.zeros(4))
    with pytest.raises(AssertionError, match="read halo before exchange"):
        ctx.x_at(3)
    ctx.halo_x = np.array([10.0, 11.0])
    assert ctx.x_at(3) == 11.0 and ctx.x_at(5) == 1.0
    with pytest.raises(AssertionError, match="outside block and halo"):
        ctx.x_at(1)
    with pytest.raises(AssertionError, match="outside its block"):
        ctx.y_add(3, 1.0)
    ctx.y_add(7, 2.5)
    assert ctx.local_y[3] == 2.5


@pytest.mark.parametrize("args", sorted(CASES["generate"]))
def test_generate_band_skew_matches_reference(args):
    c = P.generate_band_skew(*json.loads(args))
    assert _digest(c.row, c.col, c.val) == CASES["generate"][args]


def test_generate_band_skew_errors():
    with pytest.raises(ValueError, match="bandwidth must satisfy"):
        P.generate_band_skew(5, 5)
    with pytest.raises(ValueError, match="fill must be in"):
        P.generate_band_skew(5, 2, fill=1.5)


def test_csr():
    coo = P.generate_band_skew(40, 6, 0.5, 0.25, seed=3)
    csr = P.coo_to_csr(coo)
    assert np.array_equal(csr.to_dense(), coo.to_dense()) and csr.nnz == coo.nnz
    with pytest.raises(P.StructuralError, match="strictly increasing"):
        P.CsrMatrix(2, [0, 2, 2], [1, 1], [1.0, 2.0])
    with pytest.raises(P.StructuralError, match="n \\+ 1 entries"):
        P.CsrMatrix(2, [0, 1], [0], [1.0])
