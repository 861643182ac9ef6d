#!/bin/bash
# GPU box: variant sweep (attention launch-time L2 warm-up; MSS pass-L unroll). Profiling only.
TAG=${1:-r2b_var}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
for rep in 1 2; do
for lib in base warm12 warm24; do
  if [ $lib = base ]; then L=""; else L="RS_CORE_LIB=$V/$lib/librlhfspec_core.so"; fi
  env $L timeout 200 python tools/attn_bench.py c2 --layers 16 --reps 10 >> $OUT/attn_c2.jsonl 2>> $OUT/err.log
  env $L timeout 200 python tools/attn_bench.py c3s:8 --layers 8 --reps 5 >> $OUT/attn_c3s.jsonl 2>> $OUT/err.log
done
done
for lib in base lu3 lu4; do
  if [ $lib = base ]; then L=""; else L="RS_CORE_LIB=$V/$lib/librlhfspec_core.so"; fi
  echo "$lib $(env $L timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log)" >> $OUT/mss.txt
done
for lib in base warm12 warm24; do
  if [ $lib = base ]; then L=""; else L="RS_CORE_LIB=$V/$lib/librlhfspec_core.so"; fi
  env $L timeout 300 python bench.py --config c2 --no-cpu-baseline > $OUT/bench_c2_$lib.json 2>> $OUT/err.log
done
cut -c1-200 $OUT/attn_c2.jsonl $OUT/attn_c3s.jsonl; cat $OUT/mss.txt | cut -c1-120
python tools/bench_summary.py $OUT/bench_c2_*.json | cut -c1-160
