#!/bin/bash
TAG=${1:-r2b_lazy}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
timeout 900 python -m pytest tests/test_gpu_accept_compact.py tests/test_gpu_parity.py -m gpu -x -q --timeout 400 -k "fused or mss or accept or degenerate" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for r in 1 2; do
echo "cur $(timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log)" >> $OUT/mss.txt
echo "pre $(RS_CORE_LIB=$V/pre/librlhfspec_core.so timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log)" >> $OUT/mss.txt
done
cut -c1-70 $OUT/mss.txt
