cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/debug_trr.py > gpurun_out/debug_trr.log 2>&1
echo "debug rc=$?" >> gpurun_out/debug_trr.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "variants or spmv or vcycle" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python tools/tune_kernels.py --sets base= chh32=sell_chh:32 pt2=csr_per_thread:2 pt8=csr_per_thread:8 mean64=sell_max_mean:64,sell_max_len:128 > gpurun_out/tune.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune.log
