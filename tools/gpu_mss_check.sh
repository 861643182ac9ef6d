#!/bin/bash
# GPU box: accept parity + c3s bench + ncu of the MSS accept kernel. Usage: tools/gpu_mss_check.sh <tag>
TAG=${1:-mss}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "accept or compact or mask" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 400 python bench.py --config c3s --no-cpu-baseline > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_accept -s 2 -c 1 -o $OUT/prof_accept_c3s \
    python bench.py --config c3s --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_acc.log 2>&1
ls $OUT
