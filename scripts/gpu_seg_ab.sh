#!/bin/bash
# A/B of CSR region kernel builds (scripts/libps_*.so given by name), a correctness
# check of each first (scripts/seg_check.py), optional timeline of the trace build
cd $GRAFT_REPO_ROOT
libs=""
for n in "$@"; do libs="$libs scripts/libps_$n.so"; done
for l in $libs; do timeout 200 python scripts/seg_check.py $l; done 2>&1 | grep -v "^  File\|^Trace" | tee gpurun_out/seg_check.log
python scripts/seg_ab.py $libs > gpurun_out/seg_ab.log 2>&1
grep -v "^  File\|^Trace\|_lib.check\|raise" gpurun_out/seg_ab.log
if [ -f scripts/libps_trace.so ]; then
  timeout 120 python scripts/seg_trace_run.py scripts/libps_trace.so 1048576 && python scripts/seg_trace_analyze.py | tee gpurun_out/seg_trace_1m.txt
fi
