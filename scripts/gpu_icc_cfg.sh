#!/bin/bash
# instruction-cache pressure of the production kernels: icc misses and no-instruction stalls
cd $GRAFT_REPO_ROOT
for c in cfg2 cfg5 cfg1 cfg4; do
  timeout 300 ncu --clock-control none --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,sm__icc_requests.sum,sm__icc_requests_lookup_miss.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active -k regex:"scan_stream_kernel|scan_rows" -s 4 -c 1 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | grep -E "scan_|icc|no_instruction|duration|inst_executed|issue_active|pipe_" > gpurun_out/icc_$c.txt
  echo "== $c"; cat gpurun_out/icc_$c.txt
done
