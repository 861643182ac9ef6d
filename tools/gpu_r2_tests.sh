#!/bin/bash
# GPU box: the full GPU test suite + smoke (round 2). Usage: tools/gpu_r2_tests.sh <tag> [pytest -k expr]
TAG=${1:-r2tests}; OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 $K > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
tail -3 $OUT/pytest_gpu.log; tail -1 $OUT/smoke.log
