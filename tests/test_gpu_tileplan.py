"""The tile plan built on the device (csrc/tileplan_gpu.cu) against the host
builder (csrc/tileplan.cpp): tiles, windows, slice offsets and slice records
byte for byte, for every accumulator layout; plans the device builder does
not support fall back to the host builder inside pars3_plan_create."""

import ctypes

import numpy as np
import pytest

import paper_2407_17651_b200 as P
from paper_2407_17651_b200 import _lib
from paper_2407_17651_b200 import generators as G

pytestmark = pytest.mark.gpu


def _split(g, beta=None):
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    m = P.permute_sss(m0, P.rcm_order(P.pattern_from_sss(m0)))
    b = P.default_beta(m.n, P.compute_bandwidth(m)) if beta is None else beta
    return m, P.split_bands(m, b)


def _view(s):
    keep = dict(diag=np.ascontiguousarray(s.diag, np.float64), mp=np.ascontiguousarray(s.mid_ptr, np.int64),
                mc=np.ascontiguousarray(s.mid_col, np.int32), mv=np.ascontiguousarray(s.mid_val, np.float64),
                orow=np.ascontiguousarray(s.outer_row, np.int32), oc=np.ascontiguousarray(s.outer_col, np.int32),
                ov=np.ascontiguousarray(s.outer_val, np.float64))
    v = _lib.SplitView(s.n, s.beta, _lib.ptr(keep["diag"]), _lib.ptr(keep["mp"]), _lib.ptr(keep["mc"]),
                       _lib.ptr(keep["mv"]), int(keep["oc"].size), _lib.ptr(keep["orow"]), _lib.ptr(keep["oc"]),
                       _lib.ptr(keep["ov"]))
    return v, keep


def plan_arrays(s, words, use_device, options=()):
    L = _lib.load()
    v, keep = _view(s)
    opts = _lib.PlanOptions(*(tuple(options) + (0, 0, 0, -1, 0, 0, 0)[len(options):]))
    sizes = np.zeros(9, dtype=np.int64)
    rc = L.pars3_tile_plan_arrays(ctypes.byref(v), ctypes.byref(opts), words, use_device, _lib.ptr(sizes),
                                  None, None, None, None, None)
    if rc != 0:
        return None
    tiles = np.zeros(int(sizes[0]) * 12, dtype=np.int32)
    wins = np.zeros(max(1, int(sizes[1])) * 4, dtype=np.int32)
    soff = np.zeros(int(sizes[2]) + 1, dtype=np.int64)
    rec = np.zeros(max(1, int(sizes[3])), dtype=np.uint8)
    ucol = np.zeros(max(1, int(sizes[8])), dtype=np.int32)
    _lib.check(L.pars3_tile_plan_arrays(ctypes.byref(v), ctypes.byref(opts), words, use_device, _lib.ptr(sizes),
                                        _lib.ptr(tiles), _lib.ptr(wins), _lib.ptr(soff), _lib.ptr(rec),
                                        _lib.ptr(ucol)))
    return dict(sizes=sizes, tiles=tiles, wins=wins[:int(sizes[1]) * 4], slice_off=soff, rec=rec[:int(sizes[3])],
                ucol=ucol[:int(sizes[8])])


def _same(a, b, what):
    for k in ("sizes", "tiles", "wins", "slice_off", "rec", "ucol"):
        assert a[k].shape == b[k].shape, (what, k, a[k].shape, b[k].shape)
        if not np.array_equal(a[k], b[k]):
            bad = np.flatnonzero(a[k] != b[k])
            raise AssertionError(f"{what}: {k} differs at {bad[:8]} ({bad.size} places): "
                                 f"{a[k][bad[:8]]} vs {b[k][bad[:8]]}")


def _graphs():
    yield "stencil27_24", G.stencil27(24, seed_perm=9, seed_val=6), None
    yield "stencil27_24_shift", G.stencil27(24, seed_perm=3, seed_val=4, alpha=0.5), None
    yield "stencil7_40", G.stencil7(40, seed_perm=5, seed_val=6), None
    yield "grid5_300", G.grid5(300, seed_perm=7, seed_val=8), None
    yield "band_nofar", G.random_band(60000, 200, 10, 0.0, seed_struct=1, seed_perm=2, seed_val=3), None
    yield "band_wide", G.random_band(50000, 900, 24, 0.0, seed_struct=4, seed_perm=5, seed_val=6), 40


@pytest.mark.parametrize("name,g,beta", list(_graphs()), ids=lambda v: v if isinstance(v, str) else "")
@pytest.mark.parametrize("words", [2, 3, 0])
def test_device_plan_equals_host_plan(name, g, beta, words, lib_built):
    m, s = _split(g, beta)
    host = plan_arrays(s, words, 0)
    dev = plan_arrays(s, words, 1)
    if dev is None:
        pytest.skip("device builder: unsupported plan (host fallback)")
    _same(dev, host, f"{name} words={words}")


@pytest.mark.parametrize("options", [(256, 0, 0, -1), (1024, 800, 0, -1), (512, 0, 4, 3), (64, 0, 0, 0)],
                         ids=["rows256", "slots800", "seg4gap3", "rows64gap0"])
def test_device_plan_options(options, lib_built):
    m, s = _split(G.stencil27(20, seed_perm=1, seed_val=2))
    host = plan_arrays(s, 2, 0, options)
    dev = plan_arrays(s, 2, 1, options)
    if dev is None:
        pytest.skip("device builder: unsupported plan (host fallback)")
    _same(dev, host, str(options))


def test_unsupported_plans_fall_back(lib_built):
    """R-MAT (list tiles, hub rows) and far entries: the device builder declines,
    pars3_plan_create uses the host builder, products stay right."""
    import torch
    for g in (G.rmat(13, 16, seed_struct=3, seed_perm=4, seed_val=5),
              G.random_band(30000, 300, 8, 0.02, seed_struct=1, seed_perm=2, seed_val=3)):
        m, s = _split(g)
        plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
        op = P.prepare(s, plan)
        assert op.stats()["built_on_device"] == 0 or op.stats()["list_tiles"] == 0
        x = np.random.default_rng(1).uniform(-1, 1, m.n)
        y = P.spmv_pars3(s, plan, x)
        ref = P.spmv_serial(m, torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.max(np.abs(y - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_plan_create_uses_device_plan(lib_built, oracle):
    """A stencil plan is built on the device and its product matches the oracle."""
    g = G.stencil27(80, seed_perm=2, seed_val=3, alpha=0.5)
    m, s = _split(g)
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
    op = P.prepare(s, plan)
    st = op.stats()
    if st["direct"]:
        pytest.skip("row-major form chosen")
    assert st["built_on_device"] == 1
    x = np.random.default_rng(2).uniform(-1, 1, m.n)
    y = P.spmv_pars3(s, plan, x)
    ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    assert oracle.rel_err(y, ref) <= 1e-12


def test_device_plan_c5(lib_built):
    """The headline plan (c5: 19 141 tiles, 2.4 GB of records): device == host."""
    g = G.make_config("c5")
    from paper_2407_17651_b200.pipeline import prepare_gpu
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    del g
    perm, m, s, bw = prepare_gpu(m0)
    del m0, m
    host = plan_arrays(s, 2, 0)
    dev = plan_arrays(s, 2, 1)
    assert dev is not None, "the device builder must support the c5 plan"
    _same(dev, host, "c5")


def test_resident_split_plan(lib_built, oracle):
    """prepare_gpu(keep_device=True): the plan is built from the device-resident
    split (pars3_plan_create_resident), same plan and product as from the host arrays."""
    from paper_2407_17651_b200.pipeline import prepare_gpu
    g = G.stencil27(80, seed_perm=4, seed_val=5, alpha=0.5)
    m0 = P.SssMatrix._trusted(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags)
    perm, m, s, bw = prepare_gpu(m0, keep_device=True)
    assert "resident_split" in s._device
    plan, _ = P.classify_conflicts(s, P.partition_rows(m.n, 1))
    op = P.prepare(s, plan)
    assert "resident_split" not in s._device  # taken by the first plan
    st = op.stats()
    assert st["built_on_device"] == 1
    perm2, m2, s2, _ = prepare_gpu(m0)
    st2 = P.prepare(s2, plan).stats()
    for k in ("tiles", "slices", "padded_slots", "entries", "windows", "device_bytes", "list_tiles"):
        assert st[k] == st2[k], k
    x = np.random.default_rng(3).uniform(-1, 1, m.n)
    y = P.spmv_pars3(s, plan, x)
    y2 = P.spmv_pars3(s2, plan, x)
    assert np.array_equal(y, y2)
    ref = oracle.spmv_serial(m.row_ptr, m.col_ind, m.off_diags, m.diags, x)
    assert oracle.rel_err(y, ref) <= 1e-12


def _full_csr(s, device):
    L = _lib.load()
    v, keep = _view(s)
    fn = L.pars3_full_csr_device if device else L.pars3_full_csr_host
    sizes = np.zeros(4, dtype=np.int64)
    _lib.check(fn(ctypes.byref(v), _lib.ptr(sizes), None, None, None, None, None, None, None))
    nep, ne, nl, nsp = (int(t) for t in sizes)
    out = dict(col=np.zeros(nep, np.int32), val=np.zeros(nep, np.float64), lane_row=np.zeros(nl, np.int32),
               lane_flags=np.zeros(nl, np.uint32), span_row=np.zeros(max(nsp, 1), np.int32),
               span_w0=np.zeros(max(nsp, 1), np.int32), span_w1=np.zeros(max(nsp, 1), np.int32))
    _lib.check(fn(ctypes.byref(v), _lib.ptr(sizes), *(_lib.ptr(out[k]) for k in
                                                      ("col", "val", "lane_row", "lane_flags", "span_row",
                                                       "span_w0", "span_w1"))))
    for k in ("span_row", "span_w0", "span_w1"):
        out[k] = out[k][:nsp]
    out["sizes"] = sizes
    return out


@pytest.mark.parametrize("name", ["rmat", "band_far", "stencil27", "grid5", "varying_diag"])
def test_device_full_csr(name, lib_built):
    """The row-major plan built on the device (csrc/fullcsr_gpu.cu) equals the
    host builder's (csrc/fullcsr.cpp) entry for entry: hub rows spanning many
    warps, empty rows (diagonal only), padding, constant and varying diagonals."""
    g = {"rmat": lambda: G.rmat(13, 16, seed_struct=7, seed_perm=8, seed_val=9),
         "band_far": lambda: G.random_band(30001, 700, 9, 0.03, seed_struct=1, seed_perm=2, seed_val=3),
         "stencil27": lambda: G.stencil27(12, seed_val=6, alpha=0.5),
         "grid5": lambda: G.grid5(30, seed_perm=7, seed_val=8),
         "varying_diag": lambda: G.rmat(11, 8, seed_struct=1, seed_perm=2, seed_val=3)}[name]()
    m, s = _split(g)
    if name == "varying_diag":
        s = P.BandSplit(s.n, s.beta, np.linspace(-1.0, 2.0, s.n), s.mid_ptr, s.mid_col, s.mid_val, s.outer_row,
                        s.outer_col, s.outer_val)
    host, dev = _full_csr(s, False), _full_csr(s, True)
    for k in host:
        assert np.array_equal(host[k], dev[k]), (name, k)
