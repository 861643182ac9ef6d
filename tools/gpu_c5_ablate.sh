#!/bin/bash
# GPU box: c5g8 attention ablations (profiling only) + per-block pipeline trace.
OUT=gpurun_out/c5abl; mkdir -p $OUT
for d in 0 1 2 4 6 16; do
  echo "dbg=$d $(RS_ATTN_DBG=$d timeout 300 python tools/kernel_times.py c5g8 4 2>&1 | tail -1)" >> $OUT/ablate.txt
done
timeout 300 python tools/attn_trace.py c5g8 > $OUT/trace_c5g8.json 2>&1
cat $OUT/ablate.txt; tail -c 3000 $OUT/trace_c5g8.json
