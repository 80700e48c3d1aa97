#!/bin/bash
# quick GPU check: parity tests (summary kept) + per-config timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "PYTEST: $(tail -1 gpurun_out/pytest_gpu.log)"; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head -5
for c in ${CONFIGS:-c5 c3 c4 c2}; do timeout 300 python tools/prof_spmv.py $c 20 2>&1 | grep -E "spmv|phase" | tail -2; done
