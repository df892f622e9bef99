cd $GRAFT_REPO_ROOT
CMD="python bench.py --config cfg3 --steps 5 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_cfg3b.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_stream -s 3 -c 1 -o gpurun_out/prof_stream_cfg3 -f $CMD > gpurun_out/ncu_full3.log 2>&1; echo "cfg3 full rc=$?"
python scripts/select_bench.py > gpurun_out/select_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:select_scatter -s 2 -c 1 -o gpurun_out/prof_select -f python scripts/select_bench.py > gpurun_out/ncu_select.log 2>&1; echo "select full rc=$?"
du -sh gpurun_out/*
