# Full-size C5 parity + timing (setup: SRQCG, Galerkin and the level-0 smoother on the GPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3400 python tools/full_configs.py --configs 5 --gpu-setup 1 --out gpurun_out/full_configs_c5.json > gpurun_out/full_configs_c5.log 2>&1
echo "full rc=$?" >> gpurun_out/full_configs_c5.log
