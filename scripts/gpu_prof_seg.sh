#!/bin/bash
# r02 evidence for the segmented / look-back family: per case a plain run, the ncu launch
# list of the same command, and a full capture of the dominant kernel exported to CSV here
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
prof() {  # name, kernel regex, skip, command...
  local name=$1 k=$2 skip=$3; shift 3
  "$@" > gpurun_out/${name}_plain.txt 2>&1 || { echo "$name plain run failed"; return; }
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${name}_launches.csv "$@" > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f -o /tmp/$name "$@" > gpurun_out/${name}_full.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  echo "$name done"
}
prof seg1m seg_stream_kernel 2 python scripts/seg_once.py 2 3 1048576
prof seg16k seg_stream_kernel 2 python scripts/seg_once.py 2 3 16384
prof seglb1m seg_scan_kernel 2 python scripts/seg_once.py 1 3 1048576
prof tiles28 scan_tiles_kernel 3 python scripts/ab_lib.py paper_2312_14874_b200/libprefixscan_b200.so cfg3 3 scan_kernel=1
python scripts/seg_bench.py > gpurun_out/seg_bench.log 2>&1; cat gpurun_out/seg_bench.log
python scripts/ab_lib.py paper_2312_14874_b200/libprefixscan_b200.so cfg3 20 scan_kernel=1 | tee gpurun_out/tiles28_time.txt
