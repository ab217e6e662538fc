#!/bin/bash
# build an A/B variant of libpgx.so with extra -D flags into ab/:
#   tools/build_variant.sh NAME -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
srcs=$(ls paper_2010_01542_b200/csrc/*.cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -Iinclude "$@" -o ab/libpgx_$name.so $srcs
echo built ab/libpgx_$name.so
