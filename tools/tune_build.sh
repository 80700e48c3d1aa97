#!/bin/bash
# Tuning builds of libpars3 with another persistent-grid shape:
#   tools/tune_build.sh NAME THREADS MIN_BLOCKS CAP MAX_SLICES
# -> paper_2407_17651_b200/_build/tune_NAME/libpars3.so (PARS3_LIB selects it)
set -e
name=$1; thr=$2; mb=$3; cap=$4; ms=$5
d=paper_2407_17651_b200/_build/tune_$name
mkdir -p $d
cd paper_2407_17651_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp"
D="-DPARS3_THREADS=$thr -DPARS3_MIN_BLOCKS=$mb -DPARS3_CAP=$cap -DPARS3_MAX_SLICES=$ms ${EXTRA_DEFS:-}"
objs=""
for f in *.cu; do nvcc $F $D -Xptxas -v -c -o ../_build/tune_$name/${f%.cu}.o $f 2> ../_build/tune_$name/${f%.cu}.ptxas.txt; objs="$objs ../_build/tune_$name/${f%.cu}.o"; done
for f in *.cpp; do g++ -O3 -fPIC -fopenmp -std=c++17 $D -c -o ../_build/tune_$name/${f%.cpp}.cpp.o $f; objs="$objs ../_build/tune_$name/${f%.cpp}.cpp.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../_build/tune_$name/libpars3.so $objs -Xcompiler -fopenmp -lgomp
grep -A2 "k_tilesILi2ELb0ELb1" ../_build/tune_$name/tiles.ptxas.txt | grep -E "registers|spill"
