#!/bin/bash
# GPU box: accept/compact parity, bench c2 with/without the children-row L2 prefetch,
# ncu --set full of the accept kernel on c3s (MSS). Usage: tools/gpu_accept_check.sh <tag>
TAG=${1:-acc}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "accept or compact or mask" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 300 python bench.py --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
RS_ACC_PF=0 timeout 300 python bench.py --no-cpu-baseline > $OUT/bench_c2_pf0.json 2> $OUT/bench_c2_pf0.err
timeout 400 python bench.py --config c3s --no-cpu-baseline > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_accept -s 2 -c 1 -o $OUT/prof_accept_c3s \
    python bench.py --config c3s --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_acc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_accept -s 2 -c 1 -o $OUT/prof_accept_c2 \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_acc2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_compact -s 2 -c 1 -o $OUT/prof_compact_c2 \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_cmp2.log 2>&1
ls $OUT
