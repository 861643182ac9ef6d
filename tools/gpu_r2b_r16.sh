#!/bin/bash
TAG=${1:-r2b_r16}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
RS_CORE_LIB=$V/r16x/librlhfspec_core.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "attention_parity or split_kv or config3s" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for n in 12 16 17 20 24 31; do
  for v in default r16x; do
    if [ $v = default ]; then L=""; else L="RS_CORE_LIB=$V/$v/librlhfspec_core.so"; fi
    env $L timeout 300 python tools/attn_bench.py c3s:$n --layers 4 --reps 3 2>>$OUT/err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n=$n $v', d['us_per_layer'], d['frac_hbm'], d['plan'].get('num_ctas'))" >> $OUT/t.txt
  done
done
cat $OUT/t.txt
