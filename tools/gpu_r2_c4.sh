#!/bin/bash
# GPU box: config 4 with reallocation at --gpus 2 (two instance processes; on a 1-GPU box they
# share it and migrate over CUDA IPC), blocking and two-stage; N=1 reference line; synccheck of
# the degenerate-residual MSS test alone. Usage: tools/gpu_r2_c4.sh <tag>
TAG=${1:-r2c4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python bench.py --config c4 --gpus 2 --steps 300 > $OUT/bench_c4_g2.json 2> $OUT/bench_c4_g2.err
timeout 900 python bench.py --config c4 --gpus 2 --steps 300 --migration two-stage > $OUT/bench_c4_g2_ts.json 2> $OUT/bench_c4_g2_ts.err
timeout 900 python bench.py --config c4 --steps 300 > $OUT/bench_c4_g1.json 2> $OUT/bench_c4_g1.err
timeout 600 compute-sanitizer --tool synccheck --print-limit 5 --log-file $OUT/san_sync_degen.log \
   python -m pytest tests -m gpu -q -p no:cacheprovider -k "degenerate" > $OUT/san_sync_degen_pytest.log 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 5 --log-file $OUT/san_sync_invalid.log \
   python -m pytest tests -m gpu -q -p no:cacheprovider -k "invalid_draft or out_of_vocabulary or mss_full" > $OUT/san_sync_invalid_pytest.log 2>&1
for f in $OUT/*.json; do echo "== $f"; head -c 3000 $f; echo; done; tail -3 $OUT/*.err | tail -20; tail -2 $OUT/san_*
