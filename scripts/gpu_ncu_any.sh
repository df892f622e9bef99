#!/bin/bash
# one full ncu capture exported to CSV on the box: gpu_ncu_any.sh <name> <kernel regex> <skip> <command...>
cd $GRAFT_REPO_ROOT
name=$1; k=$2; skip=$3; shift 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1
echo "$name rc=$?"
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page source --csv > gpurun_out/${name}_source.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page details > gpurun_out/${name}_details.txt 2>/dev/null
