cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(lscpu | head -20; nproc; free -g) > gpurun_out/host.txt 2>&1
timeout 3300 python tools/full_configs.py --configs 1 2 3 4 5 > gpurun_out/full_configs.log 2>&1
echo "full rc=$?" >> gpurun_out/full_configs.log
