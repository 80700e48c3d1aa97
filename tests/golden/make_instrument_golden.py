"""Generate tests/golden/instrument_cases.json from the reference itself:
its instrumented twins' traces (messages, stage log, tallies, y digests) on
the golden corpus, and generate_band_skew digests.  Run in the build
container (reference importable, copied to /tmp):

    cp -r /root/reference/pkg /tmp/refpkg
    PYTHONPATH=/tmp/refpkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_instrument_golden.py
"""
import hashlib
import json
import os

import numpy as np
import skewspmv as R

HERE = os.path.dirname(os.path.abspath(__file__))
NAMES = ("tiny4", "one1", "zero3", "diag6", "tridiag5", "gen16", "gen64", "gen128shift",
         "gen257dense", "gen500")


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    z = np.load(os.path.join(HERE, "corpus.npz"))
    out = {"pars3": {}, "serial": {}, "generate": {}}
    for name in NAMES:
        n = int(z[f"{name}/n"][0])
        m = R.SssMatrix(n, z[f"{name}/row_ptr"], z[f"{name}/col_ind"].astype(np.int64),
                        z[f"{name}/off_diags"], z[f"{name}/diags"])
        x = z[f"{name}/x"]
        y, ops = R.spmv_serial_instrumented(m, x)
        out["serial"][name] = {"y": digest(y), "ops": [ops.element_reads, ops.multiply_adds]}
        for beta in (1, 3):
            s = R.split_bands(m, beta)
            for p in (1, 2, 3):
                if p > max(n, 1):
                    continue
                plan, _ = R.classify_conflicts(s, R.partition_rows(n, p))
                t = R.spmv_pars3_instrumented(s, plan, x)
                out["pars3"][f"{name}/b{beta}/p{p}"] = {
                    "y": digest(t.y),
                    "messages": [[mm.target_worker, mm.target_row, mm.value.hex(), mm.source_worker,
                                  mm.source_row, mm.source_col, mm.slot] for mm in t.messages],
                    "stage_log": [list(e) for e in t.stage_log],
                    "contexts": [[c.worker_id, c.row_start, c.row_end, c.halo_lo, c.element_reads,
                                  c.multiply_adds, c.stages, len(c.outbox)] for c in t.contexts],
                    "coordinator": [t.coordinator_reads, t.coordinator_multiply_adds, t.outer_count],
                    "total": [t.total_ops().element_reads, t.total_ops().multiply_adds],
                }
    for args in ((10, 3, 0.5, 0.0, 0), (200, 17, 0.3, 0.75, 5), (50, 49, 1.0, 0.0, 9), (30, 5, 0.0, 0.0, 1)):
        c = R.generate_band_skew(*args)
        out["generate"][json.dumps(args)] = digest(c.row, c.col, c.val)
    with open(os.path.join(HERE, "instrument_cases.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
