cd $GRAFT_REPO_ROOT
timeout 300 ./scripts/sweep > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu.log | tail -30
