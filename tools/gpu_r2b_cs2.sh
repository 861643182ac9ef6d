#!/bin/bash
TAG=${1:-r2b_cs2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
for r in 1 2; do
  echo "cs  $(timeout 300 python tools/attn_bench.py c5g8 --layers 4 --reps 5 2>>$OUT/err.log | cut -c1-120)" >> $OUT/t.txt
  echo "old $(RS_CORE_LIB=$V/nosplit/librlhfspec_core.so timeout 300 python tools/attn_bench.py c5g8 --layers 4 --reps 5 2>>$OUT/err.log | cut -c1-120)" >> $OUT/t.txt
done
cat $OUT/t.txt
timeout 400 python tools/attn_trace.py c5g8 > $OUT/trace_cs.json 2>> $OUT/err.log
