#!/bin/bash
# Attention ablations (profiling only): per-layer time with parts of the kernel disabled.
# Usage (on the GPU box): tools/attn_ablate.sh <outdir> [configs...]
OUT=${1:-gpurun_out/ablate}; shift; mkdir -p $OUT
CFGS=${@:-c2}
for c in $CFGS; do
  for d in 0 1 2 4 6 7; do
    echo "cfg=$c dbg=$d $(RS_ATTN_DBG=$d timeout 300 python tools/kernel_times.py $c 8 2>&1 | tail -1)" >> $OUT/ablate.txt
  done
done
timeout 300 python tools/attn_trace.py c2 > $OUT/trace_c2.json 2>&1
