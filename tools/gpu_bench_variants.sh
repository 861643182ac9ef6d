#!/bin/bash
# GPU box: the default bench line with the product library and variants (RS_CORE_LIB).
# Usage: tools/gpu_bench_variants.sh <tag> "<bench args>" [variant ...]
TAG=$1; ARGS=$2; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python bench.py $ARGS --no-cpu-baseline > $OUT/base.json 2> $OUT/base.err
for v in "$@"; do
  RS_CORE_LIB=paper_2512_04752_b200/_variants/$v/librlhfspec_core.so timeout 600 python bench.py $ARGS --no-cpu-baseline > $OUT/$v.json 2> $OUT/$v.err
done
python - <<PY
import json, glob
for f in sorted(glob.glob("$OUT/*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    k = d["kernels"]
    print(f.split("/")[-1], d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"].get("power_w_median"), d["roofline"]["frac"], k["attention"]["ms_per_step"], k["accept"]["ms_per_step"])
PY
