"""The C ABI: libpars3.so loads and exports every symbol include/pars3.h declares
(no compute calls -- this runs without a GPU)."""

import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "pars3.h")).read()
    return sorted(set(re.findall(r"\b(pars3_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("pars3_sss_spmv_atomic", "pars3_plan_create", "pars3_plan_spmv",
                 "pars3_plan_spmv_dot", "pars3_rcm_order", "pars3_classify_conflicts",
                 "pars3_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib_built):
    import ctypes
    from paper_2407_17651_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing


def test_python_binding_covers_header(lib_built):
    from paper_2407_17651_b200 import _lib
    assert sorted(_lib.EXPORTED) == _declared()


def test_library_is_sm100a(lib_built):
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_2407_17651_b200 import _lib
    tool = shutil.which("cuobjdump")
    if tool is None:
        return
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_plumbing(lib_built):
    """A failing host call maps to the reference's exception type and message."""
    import numpy as np
    import pytest

    import paper_2407_17651_b200 as P
    m = P.SssMatrix(4, [0, 0, 1, 2, 4], [0, 1, 0, 2], [2.0, 3.0, 5.0, 1.0], np.zeros(4))
    with pytest.raises(ValueError, match="at least 1"):
        P.split_bands(m, 0)
