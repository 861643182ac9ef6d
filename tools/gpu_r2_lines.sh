#!/bin/bash
# GPU box: the other bench lines of round 2 (c2lm, c5g8, c5 at N=1, c4) and the reference arm on
# the default config. Usage: tools/gpu_r2_lines.sh <tag>
TAG=${1:-r2lines}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python bench.py --config c2lm --no-cpu-baseline > $OUT/bench_c2lm.json 2> $OUT/c2lm.err
timeout 600 python bench.py --config c5g8 --steps 20 --no-cpu-baseline > $OUT/bench_c5g8.json 2> $OUT/c5g8.err
timeout 900 python bench.py --config c5 --steps 10 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/c5.err
timeout 900 python bench.py --config c4 --steps 300 > $OUT/bench_c4.json 2> $OUT/c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_c3s.json 2> $OUT/ref.err
for f in $OUT/*.json; do echo "== $f"; head -c 600 $f; echo; done; tail -2 $OUT/*.err
