#!/bin/bash
# GPU box: ncu evidence of the final kernels at the default line's shapes (c3s, --force-n 8) and
# c2, synccheck of the MSS kernel. Usage: tools/gpu_r2_final_evidence.sh <tag>
TAG=${1:-r2fin}; OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tree_|kv_|attn|mss_|accept|lm_head|walk" -c 400 --csv \
  --log-file $OUT/launches.csv $B --force-n 8 > $OUT/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 40 -c 1 -o $OUT/prof_attn_c3s $B --force-n 8 > $OUT/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 40 -c 1 -o $OUT/prof_attn_c2 $B --config c2 > $OUT/ncu_attn2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mss_accept" -s 2 -c 1 -o $OUT/prof_accept_c3s $B --force-n 8 > $OUT/ncu_acc.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 5 --log-file $OUT/san_sync_mss.log \
   python -m pytest tests -m gpu -q -p no:cacheprovider -k "mss or degenerate or invalid_draft or out_of_vocab" > $OUT/san_sync_mss_pytest.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 --log-file $OUT/san_mem_new.log \
   python -m pytest tests -m gpu -q -p no:cacheprovider -k "mss-1000 or attention_parity or split_kv or peer_loopback or lm_head_argmax_random or single_inf" > $OUT/san_mem_new_pytest.log 2>&1
ls $OUT
