#!/bin/bash
TAG=${1:-r2b_accsw2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
for r in 1 2; do
  for v in default lu1; do
    if [ $v = default ]; then L=""; else L="RS_CORE_LIB=$V/$v/librlhfspec_core.so"; fi
    echo "mss $v $(env $L timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log | cut -c1-30)" >> $OUT/t.txt
  done
  for v in default cs4 cs16g; do
    if [ $v = default ]; then L=""; else L="RS_CORE_LIB=$V/$v/librlhfspec_core.so"; fi
    echo "greedy $v $(env $L timeout 200 python tools/accept_launch_cost.py c2 2>>$OUT/err.log)" >> $OUT/t.txt
  done
done
cat $OUT/t.txt
