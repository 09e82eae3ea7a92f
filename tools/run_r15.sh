# Full-size parity + timing with the current defaults: C1-C3, then C5 (no dump, one timed GPU solve).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export ASPAMG_NO_CACHE=1
timeout 400 python tools/full_configs.py --configs 1 2 3 --gpu-setup 1 --out gpurun_out/full_configs_e.json > gpurun_out/full_configs_e.log 2>&1
echo "c123 rc=$?" >> gpurun_out/full_configs_e.log
timeout 3150 python tools/full_configs.py --configs 5 --gpu-setup 1 --gpu-reps 1 --out gpurun_out/full_configs_e.json >> gpurun_out/full_configs_e.log 2>&1
echo "c5 rc=$?" >> gpurun_out/full_configs_e.log
