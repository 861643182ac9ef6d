#!/bin/bash
# GPU box: the non-default bench lines after session 2b (fused commit, row map).
TAG=${1:-r2b_lines}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in c2lm c5g8 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python tools/bench_summary.py $OUT/bench_c2lm.json $OUT/bench_c5g8.json $OUT/bench_c5.json | cut -c1-260
tail -c 400 $OUT/bench_ref.json
