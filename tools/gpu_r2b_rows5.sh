#!/bin/bash
TAG=${1:-r2b_rows5}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
for r in 1 2; do
for v in pre nokids norowmap alwaysq; do
echo "$v $(RS_CORE_LIB=$V/$v/librlhfspec_core.so timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log)" >> $OUT/mss.txt
done; done
cut -c1-60 $OUT/mss.txt
