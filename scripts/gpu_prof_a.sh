cd $GRAFT_REPO_ROOT
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  CMD="python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu"
  $CMD > gpurun_out/plain_$c.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv $CMD > gpurun_out/ncu_launches_$c.log 2>&1; echo "$c launches rc=$?"
done
CMD="python bench.py --config cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu"
ncu --set full --clock-control none --import-source on -k regex:scan_stream -s 3 -c 1 -o gpurun_out/prof_stream_cfg2 -f $CMD > gpurun_out/ncu_full2.log 2>&1; echo "cfg2 full rc=$?"
CMD="python bench.py --config cfg4 --steps 5 --warmup 3 --no-e2e --no-cpu"
ncu --set full --clock-control none --import-source on -k regex:scan_rows -s 3 -c 1 -o gpurun_out/prof_rows_cfg4 -f $CMD > gpurun_out/ncu_full4.log 2>&1; echo "cfg4 full rc=$?"
du -sh gpurun_out/*
