run() { f=0; for i in 1 2 3 4 5 6 7 8; do python -m pytest tests/test_gpu_parity.py -m gpu -q -k "cfg5_small and two_stage" 2>&1 | tail -1 | grep -q failed && f=$((f+1)); done; echo "$1 failures: $f / 8"; }
run "current(lb2)"
HSVD_NO_SIDE=1 run "current(lb2)+NO_SIDE"
HSVD_BIG_CLUSTER=192 run "current(lb2)+BIG192"
