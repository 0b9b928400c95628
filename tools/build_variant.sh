#!/bin/bash
# Kernel-tuning builds: recompile aggregate_sweep.cu with extra nvcc defines and
# link libtsgm_b200<suffix>.so next to the product library (load it with
# TSGM_LIB_VARIANT=<suffix>). Usage: tools/build_variant.sh <suffix> -DNAME=VALUE ...
set -e
cd "$(dirname "$0")/.."
sfx=$1; shift
L=paper_1809_07986_b200/lib
C=paper_1809_07986_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off --expt-relaxed-constexpr -Iinclude -I$C "$@" \
  -c $C/aggregate_sweep.cu -o $L/obj/aggregate_sweep$sfx.o
objs=$(ls $L/obj/*.o | grep -v "aggregate_sweep" )
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/libtsgm_b200$sfx.so $objs $L/obj/aggregate_sweep$sfx.o -lcudart -lz
