"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container only (needs /root/reference and numba):

    python tests/golden/make_golden.py [--big]

It copies /root/reference/pkg to /tmp (the reference's numba cache writes
next to its sources), imports ``skewspmv`` from there and records:

* ``corpus.npz`` -- the reference test corpus (tests/conftest.py:41-55 of
  the reference, built with the reference's own ``generate_band_skew`` and
  ``hand_matrix``): SSS arrays, RCM labels, x, serial/dense y, and for
  beta in {1, 4, bw} x p in {1, 2, 3, 4, 8} the split/plan arrays and the
  pars3 y.
* ``c1.npz`` -- BASELINE config c1 through the full reference chain
  (pattern_from_coo -> rcm_order -> apply_permutation -> coo_to_sss ->
  split_bands -> classify_conflicts -> spmv_serial / spmv_pars3).
* ``hashes.json`` -- SHA-256 of every array of the same chain for c2 (and,
  with --big, c3 and c4, which take minutes and ~15 GB in the reference).
* with --c5: the headline config c5 (n = 16.7 M, m = 216 M).  The COO route
  (pattern_from_coo's np.unique over 2m keys, coo_normalize over 2m + n
  triplets) needs ~25 min and ~70 GB here, so the chain is entered through
  the reference's own validating constructors instead (``reference_chain_direct``):
  ``AdjacencyPattern`` (reorder.py:34-63) over the symmetrised pattern,
  the reference ``rcm_order`` (reorder.py:251-286), ``SssMatrix``
  (formats.py:163-221) over the relabelled lower triangle, then the
  reference ``split_bands`` / ``classify_conflicts`` / ``spmv_serial`` /
  ``spmv_pars3``.  The two inputs that do not come from a reference
  function -- the symmetrised pattern (oracle C restatement) and the
  relabelled lower triangle (numpy restatement of apply_permutation +
  coo_to_sss below) -- are exactly the stages the COO route pins on c2-c4.

The inputs come from paper_2407_17651_b200.generators, so the GPU box
(which has no /root/reference) regenerates identical inputs from seeds.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg"
REF_COPY = "/tmp/pars3_golden_refpkg"


def import_reference():
    if not os.path.isdir(REF_COPY):
        shutil.copytree(REF_SRC, REF_COPY)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    os.environ.setdefault("NUMBA_NUM_THREADS", "8")
    sys.path.insert(0, os.path.join(REF_COPY, "src"))
    sys.path.insert(0, ROOT)
    import skewspmv
    return skewspmv


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind in "iu":
        a = a.astype(np.int64)
    return hashlib.sha256(a.tobytes()).hexdigest()


PLAN_FIELDS = ("block_start", "row_owner", "safe_start", "conflict_idx", "conflict_ptr",
               "conflict_target", "apply_order", "apply_ptr", "halo_lo")
SPLIT_FIELDS = ("mid_ptr", "mid_col", "mid_val", "outer_row", "outer_col", "outer_val", "diag")


def corpus(R):
    tiny = [(1, 0, 2.0), (2, 1, 3.0), (3, 0, 5.0), (3, 2, 1.0)]

    def hand(n, lower, alpha=0.0):
        e = []
        for i, j, v in lower:
            e += [(i, j, v), (j, i, -v)]
        if alpha:
            e += [(d, d, alpha) for d in range(n)]
        return R.coo_normalize(R.CooMatrix.from_entries(n, e))

    g = R.generate_band_skew
    return {
        "tiny4": hand(4, tiny), "one1": R.CooMatrix.from_entries(1, []),
        "zero3": R.CooMatrix.from_entries(3, []), "diag6": hand(6, [], alpha=2.5),
        "tridiag5": g(5, 1, fill=1.0, seed=5), "gen16": g(16, 3, fill=0.5, seed=11),
        "gen64": g(64, 9, fill=0.35, seed=12), "gen128shift": g(128, 14, fill=0.25, alpha=2.5, seed=13),
        "gen257dense": g(257, 256, fill=0.9, seed=14), "gen500": g(500, 21, fill=0.15, seed=15),
    }


def make_corpus(R):
    out = {}
    for name, coo in corpus(R).items():
        m = R.coo_to_sss(coo, mode="shifted")
        x = np.random.default_rng(3).uniform(-1.0, 1.0, m.n)
        out[f"{name}/n"] = np.array([m.n])
        for f in ("row_ptr", "col_ind", "off_diags", "diags"):
            out[f"{name}/{f}"] = getattr(m, f)
        out[f"{name}/x"] = x
        out[f"{name}/y_serial"] = R.spmv_serial(m, x)
        out[f"{name}/y_dense"] = R.spmv_dense(coo, x)
        out[f"{name}/rcm_forward"] = R.rcm_order(R.pattern_from_coo(coo)).forward
        bw = R.compute_bandwidth(m)
        out[f"{name}/bandwidth"] = np.array([bw])
        for beta in sorted({1, 4, max(1, bw)}):
            s = R.split_bands(m, beta)
            for f in SPLIT_FIELDS:
                out[f"{name}/b{beta}/{f}"] = getattr(s, f)
            for p in (1, 2, 3, 4, 8):
                if p > m.n:
                    continue
                plan, rep = R.classify_conflicts(s, R.partition_rows(m.n, p))
                for f in PLAN_FIELDS:
                    out[f"{name}/b{beta}/p{p}/{f}"] = getattr(plan, f)
                out[f"{name}/b{beta}/p{p}/y_pars3"] = R.spmv_pars3(s, plan, x)
                out[f"{name}/b{beta}/p{p}/report"] = np.frombuffer(
                    json.dumps(rep.as_dict()).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "corpus.npz"), **out)
    print("corpus.npz", len(out), "arrays")


def reference_chain(R, cfg, ps=(1, 2, 4, 8)):
    """The full reference pipeline on a generator config; returns arrays."""
    from paper_2407_17651_b200 import generators as G
    g = G.make_config(cfg)
    r, c, v = G.lower_to_coo_entries(g)
    coo = R.coo_normalize(R.CooMatrix(g.n, r, c, v))
    mode = "shifted" if np.any(g.diags) else "strict"
    t = time.time()
    perm = R.rcm_order(R.pattern_from_coo(coo))
    m = R.coo_to_sss(R.apply_permutation(coo, perm), mode)
    bw = R.compute_bandwidth(m)
    beta = R.default_beta(m.n, bw)
    x = G.make_x(m.n, G.CONFIGS[cfg]["seed_x"])
    res = {"n": m.n, "nnz": m.nnz_offdiag, "bandwidth": bw, "beta": beta,
           "rcm_forward": perm.forward, "row_ptr": m.row_ptr, "col_ind": m.col_ind,
           "off_diags": m.off_diags, "diags": m.diags, "x": x,
           "y_serial": R.spmv_serial(m, x)}
    for b in (beta, max(1, bw)):
        s = R.split_bands(m, b)
        for f in SPLIT_FIELDS:
            res[f"b{b}/{f}"] = getattr(s, f)
        for p in ps:
            plan, _ = R.classify_conflicts(s, R.partition_rows(m.n, p))
            for f in PLAN_FIELDS:
                res[f"b{b}/p{p}/{f}"] = getattr(plan, f)
            res[f"b{b}/p{p}/y_pars3"] = R.spmv_pars3(s, plan, x)
    print(f"{cfg}: reference chain {time.time() - t:.1f}s n={m.n} m={m.nnz_offdiag} bw={bw}")
    return res


def _relabel_lower(n, row_ptr, col_ind, off_diags, diags, forward):
    """coo_to_sss(apply_permutation(coo, perm)) restated on the lower
    triangle: entry (i, c, v) moves to (f[i], f[c]); when the relabel puts
    it above the diagonal, its lower mirror (f[c], f[i]) carries -v
    (formats.py:14-18 sign convention); rows sorted by (row, col) as
    coo_normalize leaves them (formats.py:282-299)."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    a = forward[rows]
    b = forward[col_ind.astype(np.int64)]
    del rows
    swap = a < b
    hi = np.where(swap, b, a)
    lo = np.where(swap, a, b)
    val = np.where(swap, -off_diags, off_diags)
    del a, b, swap
    key = hi * n + lo
    del hi, lo
    order = np.argsort(key, kind="stable")
    key = key[order]
    val = val[order]
    del order
    new_rows = key // n
    col = key - new_rows * n
    del key
    counts = np.bincount(new_rows, minlength=n)
    del new_rows
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    dg = np.empty(n)
    dg[forward] = diags
    return rp, col, val, dg


def reference_chain_direct(R, cfg, ps=(1, 2, 4, 8)):
    """The reference chain entered through its validating constructors (see
    the module docstring); returns the arrays to hash."""
    from paper_2407_17651_b200 import generators as G
    from oracle import oracle as O
    g = G.make_config(cfg)
    t = time.time()
    ip, ix = O.pattern_from_sss(g.n, g.row_ptr, g.col_ind)
    pat = R.AdjacencyPattern(g.n, ip, ix)  # reorder.py:34-63 validates
    del ip, ix
    perm = R.rcm_order(pat)
    del pat
    print(f"{cfg}: reference rcm_order {time.time() - t:.1f}s", flush=True)
    rp, ci, od, dg = _relabel_lower(g.n, g.row_ptr, g.col_ind, g.off_diags, g.diags, perm.forward)
    mode_alpha = float(g.diags[0]) if g.n else 0.0
    del g
    m = R.SssMatrix(len(rp) - 1, rp, ci, od, dg)  # formats.py:163-221 validates
    del rp, ci, od, dg
    assert np.all(m.diags == mode_alpha)
    bw = R.compute_bandwidth(m)
    beta = R.default_beta(m.n, bw)
    x = G.make_x(m.n, G.CONFIGS[cfg]["seed_x"])
    res = {"n": m.n, "nnz": m.nnz_offdiag, "bandwidth": bw, "beta": beta,
           "rcm_forward": perm.forward, "row_ptr": m.row_ptr, "col_ind": m.col_ind,
           "off_diags": m.off_diags, "diags": m.diags, "x": x}
    y = R.spmv_serial(m, x)
    res["y_serial"] = y
    res["y_serial_norm_inf"] = float(np.max(np.abs(y)))
    del y
    print(f"{cfg}: relabel + serial {time.time() - t:.1f}s bw={bw} beta={beta}", flush=True)
    for b, pp in ((beta, ps), (max(1, bw), (8,))):
        s = R.split_bands(m, b)
        for f in SPLIT_FIELDS:
            res[f"b{b}/{f}"] = sha(getattr(s, f))
        res[f"b{b}/middle_count"] = int(s.mid_col.size)
        for p in pp:
            plan, _ = R.classify_conflicts(s, R.partition_rows(m.n, p))
            for f in PLAN_FIELDS:
                res[f"b{b}/p{p}/{f}"] = sha(getattr(plan, f))
            if p == 8:
                res[f"b{b}/p{p}/y_pars3"] = sha(R.spmv_pars3(s, plan, x))
            del plan
        del s
        print(f"{cfg}: beta={b} split/classify/pars3 {time.time() - t:.1f}s", flush=True)
    return res


def main():
    R = import_reference()
    hashes = {}
    path = os.path.join(HERE, "hashes.json")
    if os.path.exists(path):
        hashes = json.load(open(path))
    if "--c5" not in sys.argv:
        make_corpus(R)
        c1 = reference_chain(R, "c1")
        np.savez_compressed(os.path.join(HERE, "c1.npz"),
                            **{k: np.asarray(v) for k, v in c1.items()})
    if "--c5" in sys.argv:  # only the headline config (see the module docstring)
        res = reference_chain_direct(R, "c5")
        hashes["c5"] = {k: (sha(v) if isinstance(v, np.ndarray) else v) for k, v in res.items()}
        hashes["c5"]["route"] = "direct: AdjacencyPattern / rcm_order / SssMatrix / split_bands / classify_conflicts"
        json.dump(hashes, open(path, "w"), indent=1, sort_keys=True)
        print("hashes.json:", sorted(hashes))
        return
    cfgs = ["c2"] + (["c3", "c4"] if "--big" in sys.argv else [])
    for cfg in cfgs:
        res = reference_chain(R, cfg)
        hashes[cfg] = {k: (sha(v) if isinstance(v, np.ndarray) else v) for k, v in res.items()}
        y = res["y_serial"]
        hashes[cfg]["y_serial_norm_inf"] = float(np.max(np.abs(y)))
        json.dump(hashes, open(path, "w"), indent=1, sort_keys=True)
    print("hashes.json:", sorted(hashes))


if __name__ == "__main__":
    main()
