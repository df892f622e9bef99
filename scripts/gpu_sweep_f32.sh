#!/bin/bash
L=paper_2312_14874_b200/libprefixscan_b200.so
for le in 0 1; do for inf in 2 3 0; do for fe in 0 1; do
python scripts/ab_lib.py $L cfg2 20 stream_ledger_early=$le stream_inflight=$inf float_exact=$fe
done; done; done
python scripts/ab_lib.py $L cfg5 10
python scripts/ab_lib.py $L cfg1 50
