cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu.log | tail -8
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
for c in cfg1 cfg3 cfg4; do timeout 600 python bench.py --config $c --no-e2e --no-cpu --steps 100 > gpurun_out/bench_$c.json 2>&1; echo "$c rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', d['value']/1e9, 'Gelem/s', d['roofline']['achieved'], 'GB/s frac', d['roofline']['frac'])"; done
