cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu.log | tail -8
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
for c in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --config $c --steps 200 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', round(d['value']/1e9,1), 'Gelem/s', round(d['roofline']['achieved']), 'GB/s frac', round(d['roofline']['frac'],3), 'e2e', d['e2e'] and round(d['e2e']['value']/1e9,2), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value']/1e9,2), d['parity'])"; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
