#!/bin/bash
# Run on the GPU box (via gpurun): smoke, bench, ncu launch list of our kernels, ncu full
# captures of the attention and accept kernels. Usage: tools/gpu_bench_profile.sh <tag> [config]
set -x
TAG=${1:-r1}; CFG=${2:-c2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 900 python bench.py --config $CFG --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# launch list: every launch of our kernels over 2 timed steps (graph replays profiled per node)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tree_|kv_|attn|philox|exp_spec" \
    -c 300 --csv --log-file $OUT/launches.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 40 -c 1 -o $OUT/prof_attn \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_full_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_accept -s 2 -c 1 -o $OUT/prof_accept \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_acc_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_compact -s 2 -c 1 -o $OUT/prof_compact \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_cmp_run.log 2>&1
ls -la $OUT
