# C5 full size, call A: setup (SRQCG, Galerkin, level-0 smoother on the GPU) cached in /tmp,
# GPU solve. Meanwhile (GPU idle during the host smoother setup) the rseg tune sweep.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
df -h /tmp > gpurun_out/df.txt 2>&1
export ASPAMG_CACHE_DIR=/tmp/aspamg_cache
(sleep 420; bash tools/run_r7.sh) &
timeout 3000 python tools/full_configs.py --configs 5 --gpu-setup 1 --oracle 0 --out gpurun_out/full_configs_c5.json > gpurun_out/full_configs_c5a.log 2>&1
echo "c5a rc=$?" >> gpurun_out/full_configs_c5a.log
ls -la /tmp/aspamg_cache >> gpurun_out/df.txt
wait
