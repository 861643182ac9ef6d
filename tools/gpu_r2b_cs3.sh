#!/bin/bash
TAG=${1:-r2b_cs3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "attention" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for r in 1 2; do
  python tools/attn_bench.py c5g8 --layers 4 --reps 5 2>>$OUT/err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['us_per_layer'])" >> $OUT/t.txt
  RS_CORE_LIB=$V/split/librlhfspec_core.so python tools/attn_bench.py c5g8 --layers 4 --reps 5 2>>$OUT/err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split', d['us_per_layer'])" >> $OUT/t.txt
done
cat $OUT/t.txt
