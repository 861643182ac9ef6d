#!/bin/bash
# GPU box: dual-tile attention ablations, exp-emulation variants and trace (c5g8).
OUT=gpurun_out/dual2; mkdir -p $OUT
for d in 0 2 4 16; do
  echo "dbg=$d $(RS_ATTN_DBG=$d timeout 200 python tools/kernel_times.py c5g8 4 2>&1 | tail -1)" >> $OUT/ablate.txt
done
for v in emu2 emu3; do
  echo "$v $(RS_CORE_LIB=paper_2512_04752_b200/_variants/$v/librlhfspec_core.so timeout 200 python tools/kernel_times.py c5g8 4 2>&1 | tail -1)" >> $OUT/ablate.txt
done
timeout 200 python tools/attn_trace.py c5g8 > $OUT/trace.json 2>&1
cat $OUT/ablate.txt | cut -c1-40,180-260
python -c "
import json;d=json.load(open('$OUT/trace.json'))
for k in ('median_cycles','inflight_mean','cycles_per_block_per_cta_median','globaltimer_us'): print(k, d.get(k))
"
