#!/bin/bash
TAG=${1:-r2mss}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 -k "accept or tree_select or exp_spec" > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 200 python tools/mss_bench.py 30 > $OUT/mss_bench.json 2> $OUT/mss_bench.err
if [ -n "$2" ]; then timeout 600 ncu --set full --import-source on --clock-control none -k regex:mss_accept -c 1 -o $OUT/mss_full python tools/mss_bench.py 1 > $OUT/ncu.log 2>&1; fi
tail -3 $OUT/pytest_gpu.log; cat $OUT/mss_bench.json
