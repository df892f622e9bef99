#!/bin/bash
# round-2 session-2 check of the restored tree: GPU suite, smoke, default bench (cfg5), reference arm, cfg2
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02b_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/r02b_b5.json 2> gpurun_out/r02b_b5.err; echo "bench rc=$?"; cat gpurun_out/r02b_b5.json
python bench.py --impl reference > gpurun_out/r02b_ref5.json 2> gpurun_out/r02b_ref5.err; echo "ref rc=$?"; cat gpurun_out/r02b_ref5.json
python bench.py --config cfg2 > gpurun_out/r02b_b2.json 2> gpurun_out/r02b_b2.err; echo "cfg2 rc=$?"
