#!/bin/bash
# GPU box: the full GPU suite + smoke, then the default bench line (with the f2 sampling variant).
TAG=${1:-r2b_final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
python tools/bench_summary.py $OUT/bench_c3s.json | cut -c1-250
python -c "
import json; d=json.loads(open('$OUT/bench_c3s.json').read().strip().splitlines()[-1]); print(json.dumps(d.get('lm_head_variant')))"
bash tools/gpu_r2_tests.sh $TAG
