cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/b_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu-launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:scan_rounds -s 3 -c 1 -o gpurun_out/prof_rounds_cfg2 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"; tail -3 gpurun_out/ncu_full.log
