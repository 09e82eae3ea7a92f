cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_setup.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python tools/tune_kernels.py --sets base= u83=sell_u:83 chh8=sell_chh:8 > gpurun_out/tune.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune.log
timeout 900 python tools/setup_timing.py --configs 2,3 --out gpurun_out/setup_timing.json > gpurun_out/setup_timing.log 2>&1
echo "timing rc=$?" >> gpurun_out/setup_timing.log
