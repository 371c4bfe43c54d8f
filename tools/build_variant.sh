#!/bin/bash
# Build an alternative libwlp_b200.so with extra nvcc flags into tools/_variants/NAME.so
# (for tools/ab_variants.sh):  bash tools/build_variant.sh NAME -DWLP_MM1_MINB=3 ...
name=$1; shift
mkdir -p tools/_variants
C=paper_1501_01405_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  "$@" -shared $C/kernels.cu $C/uniforms.cu $C/ir_interp.cu $C/ir_jit.cu $C/runtime.cu -o tools/_variants/$name.so -ldl
