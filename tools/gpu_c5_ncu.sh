#!/bin/bash
# GPU box: one ncu --set full capture of the c5g8 attention kernel (tensor-bound case) + source page.
OUT=gpurun_out/c5ncu; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 90 -c 1 -o $OUT/prof_attn_c5 \
    python bench.py --config c5g8 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_run.log 2>&1
ncu -i $OUT/prof_attn_c5.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i $OUT/prof_attn_c5.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ls -la $OUT
