#!/bin/bash
# Build an experimental variant of the library (profiling only): tools/build_variant.sh <name> <nvcc -D flags...>
# Output: paper_2512_04752_b200/_variants/<name>/librlhfspec_core.so (same sources, extra -D flags).
set -e
NAME=$1; shift
cd "$(dirname "$0")/.."
OUT=paper_2512_04752_b200/_variants/$NAME; mkdir -p $OUT/obj
NCCL_INC=$(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'include'))")
NCCL_LIB=$(python -c "import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],'lib'))")
FL="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2512_04752_b200/csrc --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -I$NCCL_INC -DRS_HAVE_NCCL=1 $@"
OBJS=""
for f in paper_2512_04752_b200/csrc/*.cu paper_2512_04752_b200/csrc/*.cpp; do
  o=$OUT/obj/$(basename $f).o; /usr/local/cuda/bin/nvcc $FL -c $f -o $o & OBJS="$OBJS $o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/librlhfspec_core.so $OBJS -cudart static -L$NCCL_LIB -l:libnccl.so.2 -Xlinker -rpath=$NCCL_LIB
echo built $OUT
