#!/bin/bash
# GPU box: evidence for the session-2b kernels. Usage: tools/gpu_r2b_evidence.sh <tag>
#  - default bench line (c3s, calibrated) and c2 line
#  - ncu launch list of the default bench at fixed shapes (--force-n 8)
#  - ncu --set full of the fused MSS acceptance (c3s) and the fused greedy acceptance (c2)
#  - compute-sanitizer memcheck / racecheck / synccheck over the fused + row-map tests
TAG=${1:-r2b_ev}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_c3s.json 2> $OUT/bench_c3s.err
timeout 300 python bench.py --config c2 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tree_|kv_|attn|mss_|accept|lm_head|walk" -c 400 --csv \
  --log-file $OUT/launches.csv $B --force-n 8 > $OUT/ncu_launch_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mss_accept" -s 2 -c 1 -o $OUT/prof_accept_c3s $B --force-n 8 > $OUT/ncu_acc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tree_accept" -s 2 -c 1 -o $OUT/prof_accept_c2 $B --config c2 > $OUT/ncu_acc2.log 2>&1
K="fused or row_map or leaf"
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 --log-file $OUT/san_mem.log \
   python -m pytest tests/test_gpu_accept_compact.py -m gpu -q -p no:cacheprovider -k "not full" > $OUT/san_mem_pytest.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 --log-file $OUT/san_race.log \
   python -m pytest tests/test_gpu_accept_compact.py -m gpu -q -p no:cacheprovider -k "not full" > $OUT/san_race_pytest.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 5 --log-file $OUT/san_sync.log \
   python -m pytest tests/test_gpu_accept_compact.py -m gpu -q -p no:cacheprovider -k "not full" > $OUT/san_sync_pytest.log 2>&1
python tools/bench_summary.py $OUT/bench_c3s.json $OUT/bench_c2.json | cut -c1-300
tail -n 2 $OUT/san_*.log; tail -n 1 $OUT/san_*_pytest.log
ls $OUT
