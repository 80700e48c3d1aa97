#!/bin/bash
# DRAM bytes and duration of the product's kernels under several knob settings
# (ncu, caches not flushed between kernels):  tools/ncu_dram.sh c5 "A=1 B=2" "C=3"
cfg=$1; shift
for st in "$@"; do
  echo "== [$st]"
  env $st ncu --cache-control none --clock-control none -k regex:"k_tiles|k_conv|k_csr|k_far" -s ${SKIP:-8} -c ${COUNT:-4} \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum \
    python tools/prof_spmv.py $cfg 4 2>&1 | grep -E "k_tiles|k_conv|k_csr|dram__bytes|gpu__time|lts__t" | sed "s/  */ /g"
done
