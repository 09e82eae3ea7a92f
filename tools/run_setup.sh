cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_setup.py tests/test_cli.py -q -m gpu > gpurun_out/pytest_setup.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_setup.log
timeout 900 python tools/setup_timing.py --configs 2,3 --out gpurun_out/setup_timing.json > gpurun_out/setup_timing.log 2>&1
echo "timing rc=$?" >> gpurun_out/setup_timing.log
