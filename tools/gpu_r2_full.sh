#!/bin/bash
# GPU box, round 2: GPU tests, smoke, default bench line (c3s), c2 line, launch list of the default bench.
# Usage: tools/gpu_r2_full.sh <tag>
TAG=${1:-r2full}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
nproc > $OUT/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 400 python bench.py --config c2 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tree_|kv_|attn|mss_|accept|lm_head|walk" -c 400 --csv --log-file $OUT/launches_default.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --force-n 8 > $OUT/ncu_bench.log 2>&1
tail -3 $OUT/pytest_gpu.log; tail -1 $OUT/smoke.log; cat $OUT/bench_default.json $OUT/bench_c2.json
