#!/bin/bash
# full ncu captures of the segmented / look-back kernels, exported to CSV on the box
# (the .ncu-rep files are too large to travel back together)
cd $GRAFT_REPO_ROOT
cap() {  # name, kernel regex, skip, command...
  local name=$1 k=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1
  echo "$name rc=$?"
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv > gpurun_out/${name}_source.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
}
cap seg_stream_full seg_stream_kernel 2 python scripts/seg_once.py 2 3
cap seg_lookback_full seg_scan_kernel 2 python scripts/seg_once.py 1 3
cap tiles_full scan_tiles_kernel 3 python scripts/ab_lib.py paper_2312_14874_b200/libprefixscan_b200.so cfg3 3 scan_kernel=1
ls -la gpurun_out/
