#!/bin/bash
# A/B of several library builds: scripts/gpu_ab_multi.sh "<cfgs>" lib1.so lib2.so ...
CFGS=$1; shift
for c in $CFGS; do for rep in 1 2; do for lib in "$@"; do
  python scripts/ab_lib.py $lib $c 20
done; done; done
