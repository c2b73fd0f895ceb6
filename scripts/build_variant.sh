#!/bin/bash
# build libvpfv with extra nvcc flags into exp/libvpfv_NAME.so (A/B experiments;
# select at run time with VPFV_LIB=exp/libvpfv_NAME.so)
# usage: scripts/build_variant.sh NAME [nvcc flags...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -Iinclude "$@" \
    paper_2410_12155_b200/csrc/*.cu -o exp/libvpfv_$name.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude "$@" -Xptxas -v -c \
    paper_2410_12155_b200/csrc/stage2d2v_tma.cu -o /tmp/variant_$name.o 2>&1 | grep -A2 rb_kernel | tail -2
