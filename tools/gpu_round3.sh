#!/bin/bash
# One GPU session (round 2, re-validation): GPU tests, one bench line per
# config, the ncu launch list of the c5 product and full captures of the
# dominant kernel of c5, c4 and c3 (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/configs.jsonl
for c in c5 c4 c3 c2; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 >> gpurun_out/configs.jsonl 2> gpurun_out/configs_$c.log
  echo "$c rc=$?"
done
cat gpurun_out/configs.jsonl
timeout 300 python tools/prof_spmv.py c5 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/prof_spmv.py c5 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for c in ${FULL:-c5 c4 c3}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tiles|k_conv|k_csr" -s 4 -c 2 -o gpurun_out/full_$c python tools/prof_spmv.py $c 3 > gpurun_out/ncu_full_$c.log 2>&1; echo "ncu full $c rc=$?"
done
