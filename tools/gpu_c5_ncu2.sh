#!/bin/bash
# GPU box: ncu --set full of the c5g8 attention (dual items) + the c5g8 launch list.
OUT=gpurun_out/c5ncu2; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 90 -c 1 -o $OUT/prof_attn \
    python bench.py --config c5g8 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_run.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tree_|kv_|attn|lm_head|greedy_walk" \
    -c 200 --csv --log-file $OUT/launches.csv \
    python bench.py --config c5g8 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_launch_run.log 2>&1
ls -la $OUT
