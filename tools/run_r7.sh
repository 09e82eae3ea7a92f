# Row-segment CSR kernel (k_rseg) + 8-load CSR rounds: bit-exactness tests, then a tune sweep on C2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "rseg or variants or every_operand" > gpurun_out/pytest_r7.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r7.log
timeout 1500 python tools/tune_kernels.py --sets base= rseg1=rseg:1 rseg2=rseg:2 rseg2u83=rseg:2,rseg_u:83 rseg2u162=rseg:2,rseg_u:162 rseg2u46=rseg:2,rseg_u:46 u8=csr_u8:1 keep128=keep_bytes:134217728 > gpurun_out/tune_r7.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune_r7.log
