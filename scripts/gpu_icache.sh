#!/bin/bash
cd $GRAFT_REPO_ROOT
ncu --query-metrics 2>/dev/null | grep -i -E "icc|icache|inst_cache|l0|no_instruction|gcc" | head -40 > gpurun_out/icc_metrics.txt
for n in "$@"; do
  timeout 200 ncu --clock-control none --section WarpStateStats --section SchedulerStats --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,sm__icc_requests.sum,sm__icc_requests_lookup_miss.sum,sm__icc_requests_lookup_hit.sum -k regex:seg_stream_kernel -s 2 -c 1 python scripts/seg_trace_run.py scripts/libps_$n.so 1048576 > gpurun_out/icc_$n.txt 2>&1
done
