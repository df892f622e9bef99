cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x --timeout 600 -k "both_scan_kernels or rounds or cfg" > gpurun_out/pytest_rounds.log 2>&1; echo "pytest-rounds rc=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/pytest_rounds.log | head -5
done
