#!/bin/bash
# build_variant.sh NAME "FLAGS": the library with tmg_tweedleg.cu compiled
# with extra FLAGS, as paper_2110_08389_b200/libtmg_b200_NAME.so (A/B runs
# through TMG_LIB_PATH)
set -e
cd "$(dirname "$0")/../paper_2110_08389_b200/csrc"
make -s all >/dev/null
mkdir -p build_v
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr"
$NV $2 -c tmg_tweedleg.cu -o build_v/tmg_tweedleg_$1.o 2> build_v/$1.ptxas.log
OBJS=$(ls build/*.o | grep -v tmg_tweedleg.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libtmg_b200_$1.so $OBJS build_v/tmg_tweedleg_$1.o
grep -A2 "leg_sweep" build_v/$1.ptxas.log | grep -E "spill|registers" | tr '\n' ' '; echo " [$1]"
