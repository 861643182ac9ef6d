#!/bin/bash
# GPU box: MSS / exp_spec / fused-commit parity, MSS alone (c3s), ncu source profile of the MSS kernel.
TAG=${1:-r2b_mss}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_accept_compact.py tests/test_gpu_parity.py -m gpu -x -q --timeout 400 -k "fused or exp_spec or mss or accept or compact or philox" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
timeout 200 python tools/mss_bench.py 30 > $OUT/mss_bench.json 2> $OUT/mss_bench.err
cat $OUT/mss_bench.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mss_accept -c 1 -o $OUT/mss_full python tools/mss_bench.py 1 > $OUT/ncu.log 2>&1
tail -2 $OUT/ncu.log
