#!/bin/bash
# GPU box: acceptance parity (fused, row map, Z29), MSS alone, c3s line.
TAG=${1:-r2b_rows}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_accept_compact.py tests/test_gpu_parity.py -m gpu -x -q --timeout 400 -k "fused or exp_spec or mss or accept or compact or delta or greedy" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
timeout 200 python tools/mss_bench.py 30 > $OUT/mss_bench.json 2> $OUT/mss_bench.err
cat $OUT/mss_bench.json
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
python tools/bench_summary.py $OUT/bench_c3s.json
