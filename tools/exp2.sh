set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_finish -s 2 -c 1 -o gpurun_out/finish_c5 python tools/prof_spmv.py c5 3 > gpurun_out/ncu_fin.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_fin.log
