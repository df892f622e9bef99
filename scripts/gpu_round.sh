# one GPU call: GPU tests, smoke, bench lines for every config, reference arm,
# ncu launch lists (cfg1-5) and full captures of the cfg2 / cfg4 kernels
cd $GRAFT_REPO_ROOT
bash scripts/gpu_full.sh
bash scripts/gpu_prof_a.sh
