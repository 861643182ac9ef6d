#!/bin/bash
# GPU box: attention-only timings (tools/attn_bench.py) of the product library and variants.
# Usage: tools/gpu_attn_sweep.sh <tag> "<configs>" [variant ...]
TAG=$1; CFGS=$2; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in $CFGS; do
  timeout 300 python tools/attn_bench.py $c --trace >> $OUT/sweep.jsonl 2>> $OUT/sweep.err
  for v in "$@"; do
    RS_CORE_LIB=paper_2512_04752_b200/_variants/$v/librlhfspec_core.so timeout 300 python tools/attn_bench.py $c --trace >> $OUT/sweep.jsonl 2>> $OUT/sweep.err
  done
done
python - <<PY
import json
for l in open("$OUT/sweep.jsonl"):
    d = json.loads(l); t = d.get("trace_us", {})
    print(d["config"], d["lib"].split("/")[-2], d["us_per_layer"], d["frac_hbm"], "ends", t.get("end_min"), t.get("end_median"), t.get("end_max"))
PY
tail -3 $OUT/sweep.err
