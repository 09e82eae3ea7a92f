# Full-size C4 with a raised iteration cap (it needs more than the paper's 1000 at 400x400x4),
# then full-size C5 (setup: SRQCG, Galerkin, level-0 smoother on the GPU), both with the CPU oracle.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20) > gpurun_out/host.txt 2>&1
timeout 1500 python tools/full_configs.py --configs 4 --max-it 4000 --gpu-setup 1 --out gpurun_out/full_configs_c4.json > gpurun_out/full_configs_c4.log 2>&1
echo "c4 rc=$?" >> gpurun_out/full_configs_c4.log
timeout 3000 python tools/full_configs.py --configs 5 --gpu-setup 1 --out gpurun_out/full_configs_c5.json > gpurun_out/full_configs_c5.log 2>&1
echo "c5 rc=$?" >> gpurun_out/full_configs_c5.log
