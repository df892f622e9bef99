cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_stress_gpu.py tests/test_parity_gpu.py -q -x --timeout 600 > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/pytest_k.log | head -5
for c in cfg1 cfg2 cfg3 cfg5; do python bench.py --config $c --steps 50 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$c\", round(d[\"roofline\"][\"achieved\"]), round(d[\"roofline\"][\"frac\"],3), d[\"roofline\"][\"kernel\"][:40], d[\"parity\"])"; done
