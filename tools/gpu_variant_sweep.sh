#!/bin/bash
# Time attention per layer for each built variant (tools/build_variant.sh); profiling only.
OUT=gpurun_out/$1; mkdir -p $OUT; shift
CFGS=${CFGS:-c2}
for v in "$@"; do
  for c in $CFGS; do
    r=$(RS_CORE_LIB=paper_2512_04752_b200/_variants/$v/librlhfspec_core.so timeout 300 python tools/kernel_times.py $c 8 2>&1 | tail -1)
    echo "$v $c $(echo $r | python -c 'import sys,json
t=sys.stdin.read()
try: d=json.loads(t); print(round(d["attention_us_per_layer"],2))
except Exception: print(t[-200:])')" >> $OUT/variants.txt
  done
done
