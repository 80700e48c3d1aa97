set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "direct_mode or locality" 2>&1 | tail -3
timeout 300 python tools/det_check.py c2 c4 2>&1 | grep -v built
for v in "" ; do python tools/prof_spmv.py c4 20 2>&1 | grep -E "spmv"; done
