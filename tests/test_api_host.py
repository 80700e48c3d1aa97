"""Host-side API behaviour, mirrored from the reference's own unit tests:
formats (test_formats.py), split/partition (test_split.py), reorder
(test_reorder.py) and the error contracts (parallel.py:123-133).  No GPU."""

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from paper_2407_17651_b200.formats import DiagonalError, SkewSymmetryError, StructuralError

TINY4_LOWER = [(1, 0, 2.0), (2, 1, 3.0), (3, 0, 5.0), (3, 2, 1.0)]


def hand(n, lower, alpha=0.0):
    e = []
    for i, j, v in lower:
        e += [(i, j, v), (j, i, -v)]
    if alpha:
        e += [(d, d, alpha) for d in range(n)]
    return P.coo_normalize(P.CooMatrix.from_entries(n, e))


# ---------------------------------------------------------------- formats

def test_coo_bounds_and_lengths():
    with pytest.raises(StructuralError):
        P.CooMatrix.from_entries(2, [(0, 2, 1.0)])
    with pytest.raises(StructuralError):
        P.CooMatrix(2, np.array([0, 1]), np.array([0]), np.array([1.0]))
    with pytest.raises(StructuralError):
        P.CooMatrix.from_entries(-1, [])


def test_normalize_sums_duplicates_keeps_zero():
    m = P.CooMatrix.from_entries(3, [(2, 1, 4.0), (0, 1, 1.0), (2, 1, -1.0), (0, 0, 0.5)])
    assert list(P.coo_normalize(m).entries()) == [(0, 0, 0.5), (0, 1, 1.0), (2, 1, 3.0)]
    z = P.coo_normalize(P.CooMatrix.from_entries(2, [(1, 0, 2.0), (1, 0, -2.0)]))
    assert list(z.entries()) == [(1, 0, 0.0)]


def test_coo_to_sss_worked_example_and_modes():
    s = P.coo_to_sss(hand(4, TINY4_LOWER))
    assert s.row_ptr.tolist() == [0, 0, 1, 2, 4]
    assert s.col_ind.tolist() == [0, 1, 0, 2]
    assert s.off_diags.tolist() == [2.0, 3.0, 5.0, 1.0]
    assert s.diags.tolist() == [0.0] * 4
    sh = P.coo_to_sss(hand(4, TINY4_LOWER, alpha=2.5), mode="shifted")
    assert sh.diags.tolist() == [2.5] * 4
    with pytest.raises(DiagonalError):
        P.coo_to_sss(hand(4, TINY4_LOWER, alpha=2.5), mode="strict")
    with pytest.raises(ValueError):
        P.coo_to_sss(hand(4, TINY4_LOWER), mode="other")


def test_coo_to_sss_rejects_asymmetry_and_skew_violation():
    with pytest.raises(StructuralError):
        P.coo_to_sss(P.CooMatrix.from_entries(3, [(1, 0, 1.0)]))
    with pytest.raises(SkewSymmetryError):
        P.coo_to_sss(P.CooMatrix.from_entries(2, [(1, 0, 1.0), (0, 1, 1.0)]))


def test_sss_to_coo_round_trip_bit_exact():
    s = P.coo_to_sss(hand(4, TINY4_LOWER, alpha=2.5), mode="shifted")
    back = P.coo_to_sss(P.sss_to_coo(s), mode="shifted")
    assert back.equals(s)
    assert P.sss_to_coo(s).nnz == 12


def test_sss_validation():
    with pytest.raises(StructuralError):
        P.SssMatrix(2, [0, 1, 1], [1], [1.0], [0.0, 0.0])  # col not below row
    with pytest.raises(StructuralError):
        P.SssMatrix(3, [0, 0, 0, 2], [1, 1], [1.0, 1.0], np.zeros(3))  # not increasing
    with pytest.raises(StructuralError):
        P.SssMatrix(2, [0, 0], [], [], [0.0, 0.0])  # row_ptr length


def test_validate_skew_reports():
    rep = P.validate_skew(hand(4, TINY4_LOWER))
    assert rep.valid and rep.diagonal_class == "zero"
    bad = P.validate_skew(P.CooMatrix.from_entries(2, [(1, 0, 1.0), (0, 1, 1.0)]))
    assert not bad.valid and bad.violation_count == 1


def test_as_vector():
    assert P.as_vector([1, 2], 2).dtype == np.float64
    with pytest.raises(ValueError):
        P.as_vector(np.ones(3), 2)


def test_count_ops_worked_example():
    s = P.coo_to_sss(hand(4, TINY4_LOWER))
    assert P.count_ops(s) == P.OpCounter(element_reads=8, multiply_adds=12)


# ---------------------------------------------------------- split / plans

def test_split_worked_example(lib_built):
    s = P.split_bands(P.coo_to_sss(hand(4, TINY4_LOWER)), beta=2)
    mid = list(zip(s.mid_rows().tolist(), s.mid_col.tolist(), s.mid_val.tolist()))
    assert mid == [(1, 0, 2.0), (2, 1, 3.0), (3, 2, 1.0)]
    assert list(zip(s.outer_row.tolist(), s.outer_col.tolist())) == [(3, 0)]
    with pytest.raises(ValueError):
        P.split_bands(P.coo_to_sss(hand(4, TINY4_LOWER)), beta=0)


def test_partition_rows_known_answers():
    assert P.partition_rows(10, 4).tolist() == [0, 3, 6, 8, 10]
    assert P.partition_rows(30, 4).tolist() == [0, 8, 16, 23, 30]
    assert P.partition_rows(4, 4).tolist() == [0, 1, 2, 3, 4]
    with pytest.raises(ValueError):
        P.partition_rows(4, 0)
    with pytest.raises(ValueError):
        P.partition_rows(4, 5)


def test_classify_worked_example_and_rejects(lib_built):
    s = P.split_bands(P.coo_to_sss(hand(4, TINY4_LOWER)), beta=2)
    plan, rep = P.classify_conflicts(s, P.partition_rows(4, 2))
    assert plan.conflict_count == 1 and plan.conflict_target.tolist() == [0]
    assert rep.safe_per_worker == (1, 1) and rep.conflicts_per_worker == (0, 1)
    with pytest.raises(StructuralError):
        P.classify_conflicts(s, [0, 0, 4])
    with pytest.raises(StructuralError):
        P.classify_conflicts(s, [0, 1, 4])


def test_tridiagonal_seams(lib_built):
    lower = [(i, i - 1, float(i)) for i in range(1, 6)]
    s = P.split_bands(P.coo_to_sss(hand(6, lower)), 1)
    plan, rep = P.classify_conflicts(s, P.partition_rows(6, 3))
    assert s.mid_rows()[plan.conflict_idx].tolist() == [2, 4]
    assert rep.conflicts_per_worker == (0, 1, 1)


def test_default_beta_values():
    assert [P.default_beta(*a) for a in ((500, 30), (10000, 30), (10000, 4), (100, 0), (2, 1))] \
        == [8, 10, 4, 1, 1]


def test_pars3_argument_errors_before_any_device_work():
    """spmv_pars3 validates like the reference before touching a GPU."""
    m = P.coo_to_sss(hand(4, TINY4_LOWER))
    s2, s3 = P.split_bands(m, 2), P.split_bands(m, 3)
    plan, _ = P.classify_conflicts(s2, P.partition_rows(4, 2))
    with pytest.raises(ValueError):
        P.spmv_pars3(s3, plan, np.ones(4))
    with pytest.raises(ValueError):
        P.spmv_pars3(s2, plan, np.ones(4), p=3)
    with pytest.raises(ValueError):
        P.spmv_atomic(m, np.ones(4), 0)


def test_products_fail_loudly_without_a_device():
    """No CPU fallback: without CUDA the product raises instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    m = P.coo_to_sss(hand(4, TINY4_LOWER))
    s = P.split_bands(m, 2)
    plan, _ = P.classify_conflicts(s, P.partition_rows(4, 2))
    with pytest.raises(RuntimeError, match="CUDA device"):
        P.spmv_pars3(s, plan, np.ones(4))
    with pytest.raises(RuntimeError, match="CUDA device"):
        P.spmv_serial(m, np.ones(4))


# ---------------------------------------------------------------- reorder

def test_pattern_and_rcm_worked_example(lib_built):
    pat = P.pattern_from_coo(hand(4, TINY4_LOWER))
    adj = {i: sorted(pat.indices[pat.indptr[i]:pat.indptr[i + 1]].tolist()) for i in range(4)}
    assert adj == {0: [1, 3], 1: [0, 2], 2: [1, 3], 3: [0, 2]}
    perm = P.rcm_order(pat)
    assert sorted(perm.forward.tolist()) == [0, 1, 2, 3]


def test_permutation_validation():
    with pytest.raises(StructuralError):
        P.Permutation([0, 0, 1])
    with pytest.raises(StructuralError):
        P.Permutation([0, 3])
    assert P.Permutation.identity(3).inverse.tolist() == [0, 1, 2]


def test_rcm_path_graph_bandwidth_one(lib_built):
    rng = np.random.default_rng(3)
    n = 50
    lab = rng.permutation(n)
    lower = [(max(lab[i], lab[i + 1]), min(lab[i], lab[i + 1]), 1.0) for i in range(n - 1)]
    coo = hand(n, lower)
    perm = P.rcm_order(P.pattern_from_coo(coo))
    assert P.compute_bandwidth(P.apply_permutation(coo, perm)) == 1


def test_apply_permutation_mismatch():
    with pytest.raises(ValueError):
        P.apply_permutation(hand(4, TINY4_LOWER), P.Permutation.identity(3))
