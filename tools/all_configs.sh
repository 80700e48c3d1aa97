#!/bin/bash
# One bench line per BASELINE config on one GPU (c1 is the CPU-only case;
# c2 is L2-resident), collected into gpurun_out/configs.jsonl.
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for c in c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 ${EXTRA:-} >> gpurun_out/configs.jsonl 2> gpurun_out/configs_$c.log
  echo "$c rc=$?"
done
