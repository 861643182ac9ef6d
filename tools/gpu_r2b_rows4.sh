#!/bin/bash
TAG=${1:-r2b_rows4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
for r in 1 2; do
echo "cur $(timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log)" >> $OUT/mss.txt
echo "alwaysq $(RS_CORE_LIB=$V/alwaysq/librlhfspec_core.so timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log)" >> $OUT/mss.txt
echo "pre $(RS_CORE_LIB=$V/pre/librlhfspec_core.so timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log)" >> $OUT/mss.txt
done
cut -c1-60 $OUT/mss.txt
