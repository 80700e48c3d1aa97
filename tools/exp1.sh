set -u
for f in 0 32 48 64; do echo "== FIN_CTAS=$f"; PARS3_FIN_CTAS=$f timeout 300 python tools/det_check.py c5 c3 2>&1 | grep -v "built\|bench\]"; done
