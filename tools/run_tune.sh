cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tail" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python tools/tune_kernels.py --sets base= tail10k=tail_rows:10000 tail40k=tail_rows:40000 tail200k=tail_rows:200000 > gpurun_out/tune.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune.log
