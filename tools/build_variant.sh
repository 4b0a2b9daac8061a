#!/bin/bash
# build_variant.sh NAME "FLAGS" [SOURCE]: the library with SOURCE (default
# tmg_tweedleg.cu) compiled with extra FLAGS, as
# paper_2110_08389_b200/libtmg_b200_NAME.so (A/B runs through TMG_LIB_PATH)
set -e
cd "$(dirname "$0")/../paper_2110_08389_b200/csrc"
SRC=${3:-tmg_tweedleg.cu}
B=${SRC%.cu}
make -s all >/dev/null
mkdir -p build_v
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr"
$NV $2 -c $SRC -o build_v/${B}_$1.o 2> build_v/$1.ptxas.log
OBJS=$(ls build/*.o | grep -v "/$B.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libtmg_b200_$1.so $OBJS build_v/${B}_$1.o
grep -A2 "leg_sweep\|tail_kernel" build_v/$1.ptxas.log | grep -E "spill|registers" | tr '\n' ' '; echo " [$1]"
