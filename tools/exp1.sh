set -u
run() { echo "== $*"; env "$@" python tools/prof_spmv.py c5 20 2>&1 | grep -E "spmv|Error|error" | tail -2; }
run PARS3_X=0
run PARS3_LIB=paper_2407_17651_b200/_build/tune_a320/libpars3.so
run PARS3_LIB=paper_2407_17651_b200/_build/tune_a320/libpars3.so PARS3_TILE_ROWS=1536
run PARS3_LIB=paper_2407_17651_b200/_build/tune_a320/libpars3.so PARS3_TILE_ROWS=2048
run PARS3_LIB=paper_2407_17651_b200/_build/tune_a288/libpars3.so PARS3_TILE_ROWS=1536
run PARS3_X=0 PARS3_TILE_ROWS=1536
