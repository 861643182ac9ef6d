#!/bin/bash
TAG=${1:-r2b_rows6}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
for r in 1 2; do
echo "cur $(timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log)" >> $OUT/mss.txt
echo "pre $(RS_CORE_LIB=$V/pre/librlhfspec_core.so timeout 200 python tools/mss_bench.py 30 2>>$OUT/err.log)" >> $OUT/mss.txt
done
cut -c1-60 $OUT/mss.txt
timeout 900 python -m pytest tests/test_gpu_accept_compact.py tests/test_gpu_parity.py -m gpu -x -q --timeout 400 -k "fused or mss or accept or compact" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
python tools/bench_summary.py $OUT/bench_c3s.json
