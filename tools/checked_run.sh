#!/bin/bash
# The bounds-checked build (DCHECK, make checked) over the small cases and the
# GPU parity / determinism / peer tests (compute-sanitizer is not available on
# this pool).  Run under gpurun from the repo root.
mkdir -p gpurun_out/checked
export PARS3_LIB=paper_2407_17651_b200/_build/libpars3_checked.so
timeout 600 python tools/sanitize_cases.py > gpurun_out/checked/cases.log 2>&1; echo "cases rc=$?"; tail -2 gpurun_out/checked/cases.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_determinism.py tests/test_mrs.py tests/test_gpu_tileplan.py tests/test_gpu_locality.py -m gpu -q --timeout 900 -k "not c5" > gpurun_out/checked/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/checked/pytest.log
grep -c "check failed" gpurun_out/checked/*.log
