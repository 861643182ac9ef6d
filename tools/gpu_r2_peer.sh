#!/bin/bash
# GPU box: peer-memory migration tests (two processes), synccheck of the MSS kernel at V=128256,
# launch list of the default bench (c3s). Usage: tools/gpu_r2_peer.sh <tag>
TAG=${1:-r2peer}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_peer.py -q -x --timeout 300 > $OUT/pytest_peer.log 2>&1; echo "exit $?" >> $OUT/pytest_peer.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 --log-file $OUT/san_synccheck_mss.log \
   python -m pytest tests -m gpu -q -p no:cacheprovider -k "mss-128256 or mss-1000" > $OUT/san_synccheck_mss_pytest.log 2>&1
SEL="tree_mask or philox or accept_greedy_bit_exact or delta-1000 or kv_compact_bit_exact or attention_parity or split_kv_parity or tree_select_matches_oracle or ragged_and_flags or lm_head_argmax_random or walk_random or pack_unpack or upstream_kv"
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 --log-file $OUT/san_synccheck_rest.log \
   python -m pytest tests -m gpu -q -p no:cacheprovider -k "$SEL" > $OUT/san_synccheck_rest_pytest.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tree_|kv_|attn|mss_|accept|lm_head|walk" -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $OUT/ncu_bench.log 2>&1
tail -3 $OUT/pytest_peer.log; tail -3 $OUT/san_synccheck_*_pytest.log; tail -2 $OUT/san_synccheck_*.log
