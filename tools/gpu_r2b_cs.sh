#!/bin/bash
# GPU box: column-split dual softmax (config 5): parity first (bounded), then timing vs pre.
TAG=${1:-r2b_cs}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 240 -k "attention_dual or attention_parity or config5" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -4 $OUT/pytest.log
if grep -q "exit 0" $OUT/pytest.log; then
  for r in 1 2; do
    echo "cs  $(timeout 300 python tools/attn_bench.py c5g8 --layers 4 --reps 5 2>>$OUT/err.log | cut -c1-150)" >> $OUT/t.txt
    echo "pre $(RS_CORE_LIB=$V/pre/librlhfspec_core.so timeout 300 python tools/attn_bench.py c5g8 --layers 4 --reps 5 2>>$OUT/err.log | cut -c1-150)" >> $OUT/t.txt
  done
  cat $OUT/t.txt
fi
