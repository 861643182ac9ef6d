#!/bin/bash
# GPU box: dual-tile attention (RM = 4) parity + timing; every step under its own timeout.
OUT=gpurun_out/dual; mkdir -p $OUT
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "g8_T64 or g4_T64_dual" > $OUT/p1.log 2>&1; echo "exit $?" >> $OUT/p1.log
tail -3 $OUT/p1.log
if grep -q "exit 0" $OUT/p1.log; then
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "attention" > $OUT/p2.log 2>&1; echo "exit $?" >> $OUT/p2.log
  tail -3 $OUT/p2.log
  timeout 200 python tools/kernel_times.py c5g8 4 > $OUT/kt_dual.json 2>&1
  RS_ATTN_DUAL=0 timeout 200 python tools/kernel_times.py c5g8 4 > $OUT/kt_nodual.json 2>&1
  tail -1 $OUT/kt_dual.json; tail -1 $OUT/kt_nodual.json
fi
