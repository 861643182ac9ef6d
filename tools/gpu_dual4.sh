#!/bin/bash
OUT=gpurun_out/dual4; mkdir -p $OUT
timeout 180 python -m pytest tests/test_gpu_parity.py -x -q -k "g8_T64 or g4_T64_dual" > $OUT/p1.log 2>&1; echo "exit $?" >> $OUT/p1.log
tail -2 $OUT/p1.log
if grep -q "exit 0" $OUT/p1.log; then
  timeout 400 python -m pytest tests/test_gpu_parity.py -q -k "attention" > $OUT/p2.log 2>&1; echo "exit $?" >> $OUT/p2.log
  tail -2 $OUT/p2.log
  for d in 0 2 16 18; do echo "dbg=$d $(RS_ATTN_DBG=$d timeout 200 python tools/kernel_times.py c5g8 4 2>&1 | tail -1 | cut -c1-20,150-185)"; done
  RS_ATTN_DUAL=0 timeout 200 python tools/kernel_times.py c5g8 4 2>&1 | tail -1 | cut -c150-185
fi
