#!/bin/bash
# one iteration on the CSR region kernel: its tests, then the timings
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_seg_stream_gpu.py tests/test_parity_gpu.py -m gpu -q -x -k "seg" 2>&1 | tail -3
python scripts/seg_bench.py 2>&1 | tee gpurun_out/seg_bench.log
python scripts/seg_exp.py 2>&1 | tee gpurun_out/seg_exp.log
