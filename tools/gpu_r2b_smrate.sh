#!/bin/bash
# GPU box: per-SM streaming rates of the attention kernel (trace of one launch, repeated) to test
# whether the CTA end-time spread is a stable per-SM property. Profiling only.
TAG=${1:-r2b_smrate}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in 1 2 3 4; do
  timeout 200 python tools/attn_bench.py c2 --layers 4 --reps 3 --trace --dump >> $OUT/c2.jsonl 2>> $OUT/err.log
  timeout 200 python tools/attn_bench.py c3s:8 --layers 2 --reps 2 --trace --dump >> $OUT/c3s.jsonl 2>> $OUT/err.log
done
nvidia-smi -q | grep -i -A3 "Product Name\|Serial" | head -8 > $OUT/gpu.txt
wc -l $OUT/*.jsonl
