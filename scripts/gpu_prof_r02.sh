#!/bin/bash
# r02 profiles: per config a plain bench run, then the ncu launch list of the same command;
# full captures of the dominant kernel for cfg5 (headline) and cfg2, exported to CSV on the box
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in cfg5 cfg2 cfg1 cfg3 cfg4; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu"
  $CMD > gpurun_out/p_${c}_plain.json 2> gpurun_out/p_${c}_plain.err &&
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/p_${c}_launches.csv $CMD > /dev/null 2>&1
  echo "$c launches rc=$?"
done
for c in cfg5 cfg2; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu"
  ncu --set full --clock-control none --import-source on -k regex:scan_ -s 4 -c 1 -f -o /tmp/p_${c}_full $CMD > gpurun_out/p_${c}_full.log 2>&1
  ncu -i /tmp/p_${c}_full.ncu-rep --page raw --csv > gpurun_out/p_${c}_raw.csv 2>/dev/null
  echo "$c full rc=$?"
done
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 200 --no-e2e --no-cpu > gpurun_out/k_$c.json 2> gpurun_out/k_$c.err
  python -c "
import json;d=json.load(open('gpurun_out/k_$c.json'))
print('$c', round(d['value']/1e9,1), 'Gelem/s', round(d['roofline']['achieved']), 'GB/s frac', round(d['roofline']['frac'],3), d['parity']['ok'])"
done
