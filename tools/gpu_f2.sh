#!/bin/bash
# GPU box: f2 (fused LM head -> greedy acceptance) tests, bench lines, ncu launch list + full capture.
TAG=${1:-f2b}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_lm_head.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 600 python bench.py --config c2lm > $OUT/bench_c2lm.json 2> $OUT/bench_c2lm.err
timeout 600 python bench.py --config c5g8lm --steps 20 --no-cpu-baseline > $OUT/bench_c5g8lm.json 2> $OUT/bench_c5g8lm.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tree_|kv_|attn|lm_head|greedy_walk" \
    -c 300 --csv --log-file $OUT/launches.csv \
    python bench.py --config c2lm --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_launch_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lm_head_argmax_kernel -s 3 -c 1 -o $OUT/prof_lm_head \
    python bench.py --config c2lm --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_full_run.log 2>&1
ls -la $OUT
