#!/bin/bash
TAG=${1:-r2mssprof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 200 python tools/mss_bench.py 30 > $OUT/mss_bench.json 2> $OUT/mss_bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mss_accept -c 1 -o $OUT/mss_full python tools/mss_bench.py 1 > $OUT/ncu.log 2>&1
cat $OUT/mss_bench.json
