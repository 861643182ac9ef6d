#!/bin/bash
# L2-prefetch distance sweep (profiling only): RS_ATTN_DBG = pf << 8.
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "attention" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for c in ${2:-c2}; do
  for pf in 1 4 8 12 16 24 32; do
    echo "cfg=$c pf=$pf $(RS_ATTN_DBG=$((pf*256)) timeout 300 python tools/kernel_times.py $c 8 2>&1 | tail -1 | cut -c1-220)" >> $OUT/sweep.txt
  done
done
timeout 300 python tools/attn_trace.py c2 > $OUT/trace_c2.json 2>&1
