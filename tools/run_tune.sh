cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/tune_kernels.py > gpurun_out/tune.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune.log
