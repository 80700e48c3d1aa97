#!/bin/bash
# One GPU session (round 2, final validation): one bench line per config, the
# reference arm, the ncu launch list of the c5 product, DRAM traffic of the
# products with the caches not flushed between kernels, and full captures of
# the dominant kernels of c5, c4 and c3 (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for c in c5 c4 c3 c2; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 >> gpurun_out/configs.jsonl 2> gpurun_out/configs_$c.log
  echo "$c rc=$?"
done
cat gpurun_out/configs.jsonl | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"
timeout 300 python tools/prof_spmv.py c5 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/prof_spmv.py c5 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for c in c5 c4 c3; do
  SKIP=8 COUNT=4 tools/ncu_dram.sh $c "" > gpurun_out/ncu_dram_$c.txt 2>&1; echo "dram $c rc=$?"
done
for c in ${FULL:-c5 c4 c3}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tiles|k_conv|k_csr" -s 4 -c 2 -o gpurun_out/full_$c python tools/prof_spmv.py $c 3 > gpurun_out/ncu_full_$c.log 2>&1; echo "ncu full $c rc=$?"
done
