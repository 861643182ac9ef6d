#!/bin/bash
# GPU box: full GPU suite + smoke + default bench line + c2 line (session re-entry check).
TAG=${1:-r2b_base}; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_r2_tests.sh $TAG
timeout 600 python bench.py > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
timeout 300 python bench.py --config c2 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
tail -c 1500 $OUT/bench_c3s.json; tail -c 1500 $OUT/bench_c2.json
