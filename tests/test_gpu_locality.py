"""The locality order computed on the device (csrc/locality_gpu.cu) against
the host version (csrc/locality.cpp): the same labels and the same count of
dropped edges; and the plan built through it against the oracle."""

import os

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from paper_2407_17651_b200 import generators as G

pytestmark = pytest.mark.gpu


def _rcm_split(g):
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
    return m, P.split_bands(m, P.default_beta(m.n, P.compute_bandwidth(m)))


def _host(s):
    os.environ["PARS3_LOCALITY_HOST"] = "1"
    try:
        return P.locality_order(s)
    finally:
        del os.environ["PARS3_LOCALITY_HOST"]


CASES = [
    ("band_far", lambda: G.random_band(100000, 1024, 16, 0.01, seed_struct=21, seed_perm=22, seed_val=23)),
    ("band_far_small", lambda: G.random_band(20000, 300, 9, 0.03, seed_struct=1, seed_perm=2, seed_val=3)),
    ("stencil27", lambda: G.stencil27(16, seed_perm=3, seed_val=4)),
    ("grid5", lambda: G.grid5(80, seed_perm=7, seed_val=8)),
    ("rmat", lambda: G.rmat(13, 16, seed_struct=3, seed_perm=4, seed_val=5)),
]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_device_locality_equals_host(name, make, lib_built):
    import torch
    assert torch.cuda.is_available()
    os.environ["PARS3_LOCALITY_ALWAYS"] = "1"  # (keep the order even where the plan would drop it)
    try:
        m, s = _rcm_split(make())
        hperm, hdrop = _host(s)
        dperm, ddrop = P.locality_order(s)
    finally:
        del os.environ["PARS3_LOCALITY_ALWAYS"]
    assert ddrop == hdrop, name
    assert np.array_equal(dperm.forward, hperm.forward), name


def test_plan_through_device_locality(lib_built, oracle):
    import torch
    from paper_2407_17651_b200.device import operator_for_sss
    g = G.random_band(60000, 1024, 16, 0.01, seed_struct=11, seed_perm=12, seed_val=13)
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
    x = G.make_x(m.n, 9)
    ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    ys = []
    for host in (False, True):
        if host:
            os.environ["PARS3_LOCALITY_HOST"] = "1"
        try:
            op = operator_for_sss(m, options=(0, 0, 0, -1, 0, 8, 0) if not host else (0, 0, 0, -1, 0, 8, 1 << 20))
        finally:
            os.environ.pop("PARS3_LOCALITY_HOST", None)
        assert op.stats()["locality_order"] == 1
        y = op.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
        assert oracle.rel_err(y, ref) <= 1e-12
        ys.append(y)
    assert np.array_equal(ys[0], ys[1])  # the same plan either way: the same bits
