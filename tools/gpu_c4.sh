#!/bin/bash
# GPU box: config 4 generation loop tests + bench line. Usage: tools/gpu_c4.sh <tag>
TAG=${1:-c4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_instance.py -x -q > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 900 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "exit $?" >> $OUT/bench_c4.err
timeout 300 python bench.py --config c4 --impl reference --steps 3 --warmup 3 > $OUT/bench_c4_ref.json 2> $OUT/bench_c4_ref.err
ls $OUT
