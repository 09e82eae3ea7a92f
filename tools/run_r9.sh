# rseg restricted to large operands (>= 64k rows), pipelined variants; sorted SELL windows; u8 + 16-bit long rows.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "rseg" > gpurun_out/pytest_r9.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r9.log
timeout 1500 python tools/tune_kernels.py --sets base= p1044=rseg:1,rseg_u:1044 p1045=rseg:1,rseg_u:1045 p1083=rseg:1,rseg_u:1083 p1082=rseg:1,rseg_u:1082 p2_1083=rseg:2,rseg_u:1083 sort256=sell_sort:1,sell_sigma:256 u8h=csr_u8:1,idx16_max_group:256 h256=idx16_max_group:256 > gpurun_out/tune_r9.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune_r9.log
