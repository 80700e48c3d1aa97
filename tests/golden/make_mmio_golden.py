"""Generate tests/golden/mmio_cases.json: the reference reader's verdict
(result digest or exception type + message) on a set of Matrix Market,
vector and permutation texts.  Run in the build container, where the
reference is importable (copied to /tmp so numba caches stay out of it):

    cp -r /root/reference/pkg /tmp/refpkg
    PYTHONPATH=/tmp/refpkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_mmio_golden.py
"""
import hashlib
import json
import os
import tempfile

import numpy as np
import skewspmv as R

HERE = os.path.dirname(os.path.abspath(__file__))

MATRICES = {
    "general_ok": "%%MatrixMarket matrix coordinate real general\n% c\n\n3 3 4\n1 1 2.5\n2 1 -1e-3\n3 2 7\n1 3 0\n",
    "skew_ok": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 3\n2 1 0.5\n3 1 -2\n3 3 0\n",
    "sym_ok": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 4\n2 1 1.25\n",
    "dup_sum": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 2 1\n1 2 2\n2 2 -0\n",
    "upper_case_hdr": "%%MatrixMarket MATRIX Coordinate REAL General\n1 1 1\n1 1 3\n",
    "crlf": "%%MatrixMarket matrix coordinate real general\r\n2 2 1\r\n2 1 3\r\n",
    "underscore": "%%MatrixMarket matrix coordinate real general\n2 2 1\n2 1 1_000.5\n",
    "indented_comment": "%%MatrixMarket matrix coordinate real general\n2 2 1\n  % not a comment\n2 1 3\n",
    "inf_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n2 1 -inf\n",
    "empty": "",
    "bad_banner": "%MatrixMarket matrix coordinate real general\n1 1 0\n",
    "bad_object": "%%MatrixMarket vector coordinate real general\n1 1 0\n",
    "bad_format": "%%MatrixMarket matrix array real general\n1 1 0\n",
    "bad_field": "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
    "bad_qual": "%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "size_fields": "%%MatrixMarket matrix coordinate real general\n3 3\n",
    "size_nonint": "%%MatrixMarket matrix coordinate real general\n3 3 x\n",
    "not_square": "%%MatrixMarket matrix coordinate real general\n3 4 0\n",
    "neg_nnz": "%%MatrixMarket matrix coordinate real general\n3 3 -1\n",
    "entry_fields": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 2\n",
    "entry_malformed": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 2 abc\n",
    "too_many": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 2 1\n2 1 1\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n3 3 1\n4 1 1\n",
    "upper_in_skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 1\n1 2 1\n",
    "skew_diag": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 1\n2 2 1.50\n",
    "too_few": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 1\n",
    "nan_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n2 1 nan\n",
}
VECTORS = {
    "vec_ok": "1\n% c\n\n  -2.5e3\n3\n",
    "vec_bad": "1\n2 3\n",
    "vec_inf": "inf\n-Infinity\n",
}
PERMS = {
    "perm_ok": "3\n0 2\n2 0\n1 1\n",
    "perm_empty": "",
    "perm_count": "x\n",
    "perm_len": "3\n0 1\n",
    "perm_pair": "2\n0 1 2\n1 0\n",
    "perm_range": "2\n0 1\n5 0\n",
    "perm_twice": "2\n1 0\n1 1\n",
    "perm_nonint": "2\n0 a\n1 0\n",
    "perm_not_bijection": "2\n0 0\n1 0\n",
}


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def verdict(fn):
    try:
        return {"ok": fn()}
    except Exception as e:  # noqa: BLE001 - the verdict is the exception
        return {"error": type(e).__name__, "message": str(e)}


def main():
    out = {"matrix": {}, "vector": {}, "permutation": {}}
    with tempfile.TemporaryDirectory() as d:
        for group, cases, fn in (
                ("matrix", MATRICES, lambda p: (lambda r: [r[1], int(r[0].n), digest(r[0].row, r[0].col, r[0].val)])(R.read_matrix(p))),
                ("vector", VECTORS, lambda p: digest(R.read_vector(p))),
                ("permutation", PERMS, lambda p: digest(R.read_permutation(p).forward))):
            for name, text in cases.items():
                path = os.path.join(d, name)
                with open(path, "w", encoding="ascii", newline="") as fh:
                    fh.write(text)
                out[group][name] = {"text": text, **verdict(lambda: fn(path))}
    with open(os.path.join(HERE, "mmio_cases.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
