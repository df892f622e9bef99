#!/bin/bash
# A/B of two library builds over the 1-D configs (scripts/ab_lib.py)
A=paper_2312_14874_b200/libprefixscan_b200.so
B=${1:-scripts/libps_nbuf7.so}
for c in cfg1 cfg2 cfg3 cfg5; do
  for lib in $A $B $A $B; do python scripts/ab_lib.py $lib $c 20; done
done
python scripts/ab_lib.py $A cfg2 20 float_exact=1
python scripts/ab_lib.py $B cfg2 20 float_exact=1
