#!/bin/bash
# GPU box, round-2 baseline: GPU tests, smoke, bench c2 + c3s, launch list of c3s.
TAG=${1:-r2base}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 400 python bench.py --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 400 python bench.py --config c3s --no-cpu-baseline > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
ls $OUT
