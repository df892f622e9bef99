#!/bin/bash
# final evidence for the segmented path: tests, soak, bench-style lines, ncu launch lists and full captures
cd $GRAFT_REPO_ROOT
timeout 1300 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 400 python scripts/soak.py 240 2>&1 | tail -2
for s in 16384 1048576 16777216; do timeout 250 python scripts/seg_line.py --nseg $s > gpurun_out/seg_line_$s.json 2>/dev/null; done
timeout 250 python scripts/seg_line.py --no-totals > gpurun_out/seg_line_notot.json 2>/dev/null
timeout 200 python scripts/seg_dtypes.py > gpurun_out/seg_dtypes.log 2>&1; cat gpurun_out/seg_dtypes.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
prof() {
  local name=$1 k=$2 skip=$3; shift 3
  "$@" > gpurun_out/${name}_plain.txt 2>&1 || { echo "$name plain run failed"; return; }
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${name}_launches.csv "$@" > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f -o /tmp/$name "$@" > gpurun_out/${name}_full.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  echo "$name done"
}
prof seg1m seg_stream_kernel 2 python scripts/seg_once.py 2 3 1048576
prof seg16k seg_stream_kernel 2 python scripts/seg_once.py 2 3 16384
prof segf32 seg_stream_kernel 2 python scripts/seg_f32_once.py 16384 3
