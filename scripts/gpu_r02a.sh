#!/bin/bash
# round-2 first check: host pipeline tests, the cfg5 headline bench and the reference arm
set -x
python -m pytest tests/test_host_gpu.py tests/test_abi.py -x -q 2>&1 | tail -5
python bench.py > gpurun_out/r02_b5.json 2> gpurun_out/r02_b5.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02_ref5.json 2> gpurun_out/r02_ref5.err; echo "ref rc=$?"
