#!/bin/bash
TAG=${1:-r2b_emu}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
for r in 1 2; do
for v in default emu1 f2 emu1f2 emu0f2; do
  if [ $v = default ]; then L=""; else L="RS_CORE_LIB=$V/$v/librlhfspec_core.so"; fi
  env $L timeout 300 python tools/attn_bench.py c5g8 --layers 4 --reps 5 2>>$OUT/err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['us_per_layer'])" >> $OUT/t.txt
done; done
cat $OUT/t.txt
