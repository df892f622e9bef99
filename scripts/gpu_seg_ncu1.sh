#!/bin/bash
# one full ncu capture of seg_stream_kernel (2^20 segments), exported to CSV on the box
cd $GRAFT_REPO_ROOT
name=${1:-seg_stream_full}
ncu --set full --clock-control none --import-source on -k regex:seg_stream_kernel -s 2 -c 1 -f -o /tmp/$name python scripts/seg_once.py 2 3 > gpurun_out/$name.log 2>&1
echo "$name rc=$?"
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page source --csv > gpurun_out/${name}_source.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
