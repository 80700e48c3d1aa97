#!/bin/bash
# One GPU session: parity tests, the bench line, the ncu launch list and one
# full ncu capture of the tile kernel (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 200 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.log; echo "bench rc=$?"; tail -3 gpurun_out/bench.log; cat gpurun_out/bench.json
timeout 300 python tools/prof_spmv.py c5 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_spmv.py c5 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 2 -c 1 -o gpurun_out/prof_c5 python tools/prof_spmv.py c5 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
