#!/bin/bash
# Build an alternative library for scripts/ab.sh: _ab/<name>.so with one
# translation unit recompiled under extra flags.
#   scripts/mk_variant.sh wpc5 pg_walkm -DPG_WALKM_WPC_LARGE=5
cd "$(dirname $0)/../paper_1905_12146_b200/csrc"
name=$1; tu=$2; shift 2
mkdir -p ../../_ab /tmp/ab_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr "$@" -c $tu.cu -o /tmp/ab_$name/$tu.o 2> /tmp/ab_$name/$tu.ptxas.log || { tail -20 /tmp/ab_$name/$tu.ptxas.log; exit 1; }
objs=$(ls ../_build/*.o | grep -v "/$tu.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../_ab/$name.so $objs /tmp/ab_$name/$tu.o -lpthread && echo "built _ab/$name.so"
