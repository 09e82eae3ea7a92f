# C4 (thin plate) defaults check: dense tail / long-row split on and off.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/tune_kernels.py --config 4 --sets base= td0=tail_dense:0 long0=csr_long:0 both0=tail_dense:0,csr_long:0 --out gpurun_out/tune_c4.json > gpurun_out/tune_r18_c4.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune_r18_c4.log
