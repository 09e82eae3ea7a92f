# C4 full size with the current defaults: the paper's max_it 1000, then max_it 4000.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/full_configs.py --configs 4 --gpu-setup 1 --gpu-reps 1 --out gpurun_out/full_configs_c4e.json > gpurun_out/full_configs_c4e.log 2>&1
echo "c4 rc=$?" >> gpurun_out/full_configs_c4e.log
timeout 1500 python tools/full_configs.py --configs 4 --max-it 4000 --gpu-setup 1 --gpu-reps 1 --out gpurun_out/full_configs_c4e.json >> gpurun_out/full_configs_c4e.log 2>&1
echo "c4 4000 rc=$?" >> gpurun_out/full_configs_c4e.log
