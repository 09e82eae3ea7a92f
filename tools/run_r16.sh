# Vectorized 16-bit CSR kernel: parity tests, then SELL unroll / CSR sweeps on C2 (current defaults as base).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "vectorized" > gpurun_out/pytest_r16.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r16.log
timeout 1200 python tools/tune_kernels.py --sets base= vec=csr_vec:1 vecpt2=csr_vec:1,csr_per_thread:2 pt8u8=csr_per_thread:8,csr_u8:2 sell84=sell_u:84 sell83=sell_u:83 > gpurun_out/tune_r16.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune_r16.log
