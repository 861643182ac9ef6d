#!/bin/bash
# GPU box: c5g8 (tensor-bound attention) with a share of the softmax exponentials on the FMA
# pipe (variants built by tools/build_variant.sh emuN -DRS_ATTN_EXP_EMU=N). Usage: <tag>
TAG=${1:-emu}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python bench.py --config c5g8 --steps 20 --no-cpu-baseline > $OUT/c5_base.json 2> $OUT/c5_base.err
for e in 2 3 4; do
  RS_CORE_LIB=paper_2512_04752_b200/_variants/emu$e/librlhfspec_core.so timeout 300 python bench.py --config c5g8 --steps 20 --no-cpu-baseline > $OUT/c5_emu$e.json 2> $OUT/c5_emu$e.err
  RS_CORE_LIB=paper_2512_04752_b200/_variants/emu$e/librlhfspec_core.so timeout 300 python bench.py --config c2 --steps 30 --no-cpu-baseline > $OUT/c2_emu$e.json 2> $OUT/c2_emu$e.err
done
RS_CORE_LIB=paper_2512_04752_b200/_variants/emu3/librlhfspec_core.so timeout 600 python -m pytest tests -m gpu -x -q -k attention > $OUT/pytest_emu3.log 2>&1
ls $OUT
