#!/bin/bash
# build_variant.sh <name> [-DFLAG=...]...  ->  variants/libmk2_<name>.so (A/B builds; variants/ is git-ignored scratch)
name=$1; shift
mkdir -p variants
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -shared --use_fast_math "$@" \
  -o variants/libmk2_$name.so paper_1909_04750_b200/csrc/mk2_api.cu -lcudart
