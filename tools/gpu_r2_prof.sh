#!/bin/bash
# GPU box, round 2: ncu --set full captures of the current attention kernel (c3s headline and c2),
# MSS accept and compaction on c3s; compute-sanitizer memcheck/racecheck/synccheck/initcheck over
# every kernel at small sizes (selected GPU tests). Usage: tools/gpu_r2_prof.sh <tag>
TAG=${1:-r2prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 40 -c 1 -o $OUT/prof_attn_c3s \
    $B --config c3s > $OUT/ncu_attn_c3s.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 40 -c 1 -o $OUT/prof_attn_c2 \
    $B --config c2 > $OUT/ncu_attn_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mss_accept|tree_accept" -s 2 -c 1 -o $OUT/prof_accept_c3s \
    $B --config c3s > $OUT/ncu_acc_c3s.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kv_compact -s 2 -c 1 -o $OUT/prof_compact_c3s \
    $B --config c3s > $OUT/ncu_cmp_c3s.log 2>&1
SEL="tree_mask or philox or accept_greedy_bit_exact or delta-1000 or mss-1000 or degenerate or invalid_draft or out_of_vocabulary or kv_compact_bit_exact or attention_parity or split_kv_parity or tree_select_matches_oracle or ragged_and_flags or lm_head_argmax_random or walk_random or pack_unpack or upstream_kv"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 --log-file $OUT/san_$tool.log \
      python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$SEL" > $OUT/san_${tool}_pytest.log 2>&1
  echo "exit $?" >> $OUT/san_${tool}_pytest.log
done
ls $OUT; tail -2 $OUT/san_*_pytest.log; tail -3 $OUT/san_*.log
