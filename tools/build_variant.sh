#!/bin/bash
# Kernel-variant experiments: build/variants/libcvpb200_<name>.so with extra
# nvcc flags on cvp_kernels.cu and api.cpp (the other objects come from the
# main build). Load one with CVPB_LIB=build/variants/libcvpb200_<name>.so.
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2110_09841_b200/csrc"
B=../../build/csrc
O=../../build/variant_obj
mkdir -p ../../build/variants $O
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -I../../include -Xptxas -v --expt-relaxed-constexpr"
/usr/local/cuda/bin/nvcc $F "$@" -c cvp_kernels.cu -o $O/cvp_kernels_$name.o 2> $O/cvp_kernels_$name.ptxas.txt \
  || (cat $O/cvp_kernels_$name.ptxas.txt; false)
/usr/local/cuda/bin/nvcc $F "$@" -x cu -c api.cpp -o $O/api_$name.o 2> /dev/null
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o ../../build/variants/libcvpb200_$name.so \
  $O/cvp_kernels_$name.o $B/cvp_kernels_b.o $B/cvp_kernels_c.o $B/siddon_kernels.o $B/tt_kernels.o $B/vecops.o $O/api_$name.o $B/group.o $B/group_kernels.o
grep -A2 "cvp_brick_kernelILb1ELb[01]ELb1ELb1ELi2E" $O/cvp_kernels_$name.ptxas.txt | grep -E "registers|spill"
