# full ncu captures of the cfg1 and cfg3 stream kernels (after a plain run of the same command)
cd $GRAFT_REPO_ROOT
for c in cfg1 cfg3; do
  CMD="python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu"
  $CMD > gpurun_out/plain_$c.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:scan_stream -s 3 -c 1 -o gpurun_out/prof_stream_$c -f $CMD > gpurun_out/ncu_full_$c.log 2>&1; echo "$c full rc=$?"
done
