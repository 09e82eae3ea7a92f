set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
(lscpu; nproc; free -g) > gpurun_out/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
