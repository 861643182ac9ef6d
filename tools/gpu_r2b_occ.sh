#!/bin/bash
TAG=${1:-r2b_occ}; OUT=gpurun_out/$TAG; mkdir -p $OUT
V=paper_2512_04752_b200/_variants
M=launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__occupancy_per_cluster_size,launch__shared_mem_per_block_static,launch__shared_mem_per_block_dynamic,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 300 ncu --metrics $M -k regex:mss_accept -c 1 --csv python tools/mss_bench.py 1 > $OUT/cur.csv 2>&1
RS_CORE_LIB=$V/pre/librlhfspec_core.so timeout 300 ncu --metrics $M -k regex:mss_accept -c 1 --csv python tools/mss_bench.py 1 > $OUT/pre.csv 2>&1
grep -h "launch__\|gpu__time\|warps_active" $OUT/cur.csv $OUT/pre.csv | awk -F'","' '{print $(NF-2), $NF}'
