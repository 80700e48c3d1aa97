#!/bin/bash
# One GPU session (round 2): the bench line, the reference arm, the ncu
# launch list of the bench's product and one full capture of each kernel of
# the c5 product (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
CFG=${CFG:-c5}
timeout 900 python bench.py --config $CFG --steps 50 --warmup 5 > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.log; echo "bench rc=$?"; tail -4 gpurun_out/bench_$CFG.log; cat gpurun_out/bench_$CFG.json
if [ "${REF:-1}" = 1 ]; then
timeout 900 python bench.py --impl reference --config $CFG --steps 5 --warmup 3 > gpurun_out/bench_ref_$CFG.json 2> gpurun_out/bench_ref_$CFG.log; echo "ref rc=$?"; tail -3 gpurun_out/bench_ref_$CFG.log; cat gpurun_out/bench_ref_$CFG.json
fi
if [ "${NCU:-1}" = 1 ]; then
timeout 300 python tools/prof_spmv.py $CFG 3 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv python tools/prof_spmv.py $CFG 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tiles|k_finish|k_csr" -s 2 -c 2 -o gpurun_out/full_$CFG python tools/prof_spmv.py $CFG 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
