#!/bin/bash
# r02 segmented / look-back evidence: bench by segment count, hand-off timeline,
# full captures of seg_stream_kernel (2^20 segments) and scan_tiles_kernel (2^28)
cd $GRAFT_REPO_ROOT
python scripts/seg_bench.py > gpurun_out/seg_bench.log 2>&1; cat gpurun_out/seg_bench.log
python scripts/seg_exp.py > gpurun_out/seg_exp.log 2>&1; cat gpurun_out/seg_exp.log
if [ -f scripts/libps_segtrace.so ]; then
  python scripts/seg_trace_run.py scripts/libps_segtrace.so 1048576 && python scripts/seg_trace_analyze.py > gpurun_out/seg_trace_1m.txt; cat gpurun_out/seg_trace_1m.txt
  python scripts/seg_trace_run.py scripts/libps_segtrace.so 1048576 notot && python scripts/seg_trace_analyze.py > gpurun_out/seg_trace_1m_notot.txt; cat gpurun_out/seg_trace_1m_notot.txt
  python scripts/seg_trace_run.py scripts/libps_segtrace.so 16384 && python scripts/seg_trace_analyze.py > gpurun_out/seg_trace_16k.txt; cat gpurun_out/seg_trace_16k.txt
fi
python scripts/seg_once.py 2 3 && ncu --set full --clock-control none --import-source on -k regex:seg_stream_kernel -s 2 -c 1 -f -o gpurun_out/seg_stream_full python scripts/seg_once.py 2 3 > gpurun_out/seg_stream_full.log 2>&1; echo "seg full rc=$?"
python scripts/seg_once.py 1 3 && ncu --set full --clock-control none --import-source on -k regex:seg_scan_kernel -s 2 -c 1 -f -o gpurun_out/seg_lookback_full python scripts/seg_once.py 1 3 > gpurun_out/seg_lookback_full.log 2>&1; echo "seg lb full rc=$?"
python scripts/ab_lib.py paper_2312_14874_b200/libprefixscan_b200.so cfg3 10 scan_kernel=1 && ncu --set full --clock-control none --import-source on -k regex:scan_tiles_kernel -s 3 -c 1 -f -o gpurun_out/tiles_full python scripts/ab_lib.py paper_2312_14874_b200/libprefixscan_b200.so cfg3 3 scan_kernel=1 > gpurun_out/tiles_full.log 2>&1; echo "tiles full rc=$?"
