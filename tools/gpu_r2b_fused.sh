#!/bin/bash
# GPU box: fused accept + compact parity, then the c2 / c3s lines. Usage: tools/gpu_r2b_fused.sh <tag>
TAG=${1:-r2b_fused}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_accept_compact.py tests/test_gpu_parity.py -m gpu -x -q --timeout 400 -k "fused or compact or accept" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
timeout 300 python bench.py --config c2 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
python tools/bench_summary.py $OUT/bench_c2.json $OUT/bench_c3s.json
