#!/bin/bash
# GPU box: full GPU test suite, smoke, bench lines (c2 default, c3s, c4, c5g8), MSS variant.
# Usage: tools/gpu_round.sh <tag>
TAG=${1:-round}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 400 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 400 python bench.py --config c3s --no-cpu-baseline > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
timeout 600 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 400 python bench.py --config c5g8 --steps 20 --no-cpu-baseline > $OUT/bench_c5g8.json 2> $OUT/bench_c5g8.err
ls $OUT
