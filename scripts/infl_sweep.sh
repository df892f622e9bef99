# in-flight TMA region limit of the stream kernel (StreamArgs.inflight): A/B at mid sizes
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for i in 0 1 2 3; do echo "== INFL=$i"; MID=1 INFL=$i ./scripts/stream_variants; done; done
