#!/bin/bash
TAG=${1:-r2b_db}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
timeout 900 python -m pytest tests/test_gpu_accept_compact.py tests/test_gpu_parity.py -m gpu -x -q --timeout 400 -k "fused or mss or accept or degenerate or delta or greedy" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for r in 1 2 3; do
  echo "new $(timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log | cut -c1-30) $(timeout 200 python tools/accept_launch_cost.py c2 2>>$OUT/err.log | cut -c1-40)" >> $OUT/t.txt
  echo "old $(RS_CORE_LIB=$V/prev/librlhfspec_core.so timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log | cut -c1-30) $(RS_CORE_LIB=$V/prev/librlhfspec_core.so timeout 200 python tools/accept_launch_cost.py c2 2>>$OUT/err.log | cut -c1-40)" >> $OUT/t.txt
done
cat $OUT/t.txt
