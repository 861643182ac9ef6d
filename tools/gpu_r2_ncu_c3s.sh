#!/bin/bash
# GPU box: ncu evidence for the default bench line (c3s at the calibrated n = 9: T = 10): launch
# list of two timed steps, --set full of one attention launch, MSS accept and compaction.
TAG=${1:-r2ncu}; N=${2:-9}; OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 --force-n $N"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tree_|kv_|attn|mss_|accept|lm_head|walk" -c 400 --csv \
  --log-file $OUT/launches.csv $B > $OUT/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 40 -c 1 -o $OUT/prof_attn_c3s $B > $OUT/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mss_accept" -s 2 -c 1 -o $OUT/prof_accept_c3s $B > $OUT/ncu_acc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_compact -s 2 -c 1 -o $OUT/prof_compact_c3s $B > $OUT/ncu_cmp.log 2>&1
ls $OUT; tail -2 $OUT/*.log
