#!/bin/bash
TAG=${1:-r2b_lu1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
timeout 900 python -m pytest tests/test_gpu_accept_compact.py tests/test_gpu_parity.py -m gpu -x -q --timeout 400 -k "fused or mss or accept or degenerate" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for r in 1 2 3; do
  echo "lu1 $(timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log | cut -c1-30)" >> $OUT/t.txt
  echo "lu2 $(RS_CORE_LIB=$V/lu2/librlhfspec_core.so timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log | cut -c1-30)" >> $OUT/t.txt
done
cat $OUT/t.txt
timeout 900 python bench.py --no-cpu-baseline --no-lm-variant > $OUT/bench_c3s.json 2> $OUT/b.err
python tools/bench_summary.py $OUT/bench_c3s.json | cut -c1-250
