#!/bin/bash
# build library variants in parallel: scripts/build_variants.sh name1 "flags1" name2 "flags2" ...
# -> scripts/libps_<name>.so (git-ignored; they travel to the GPU box)
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC $flags \
      -o scripts/libps_$name.so paper_2312_14874_b200/csrc/prefixscan_b200.cu > /tmp/build_$name.log 2>&1; echo "$name rc=$?" ) &
done
wait
