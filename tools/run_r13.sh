# C5 full size in one call (setup without dump, one warm + one timed GPU solve, CPU oracle solve),
# recording the residual histories of both solves.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export ASPAMG_NO_CACHE=1
timeout 3500 python tools/full_configs.py --configs 5 --gpu-setup 1 --gpu-reps 1 --out gpurun_out/full_configs_c5h.json > gpurun_out/full_configs_c5h.log 2>&1
echo "c5 rc=$?" >> gpurun_out/full_configs_c5h.log
