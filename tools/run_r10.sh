# C5 full size in one call: setup (no dump), one warm + one timed GPU solve, the CPU oracle solve
# on all host cores. The GPU is idle during the host smoother setup: the r9 tune runs then.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export ASPAMG_NO_CACHE=1
(sleep 400; bash tools/run_r9.sh) &
timeout 3450 python tools/full_configs.py --configs 5 --gpu-setup 1 --gpu-reps 1 --out gpurun_out/full_configs_c5.json > gpurun_out/full_configs_c5.log 2>&1
echo "c5 rc=$?" >> gpurun_out/full_configs_c5.log
wait
