#!/bin/bash
# Round-2 GPU session E: tile-local SELL (x footprint in shared memory, 16-bit local columns) on the LONG-row operands.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
O=gpurun_out
X="xsell_min_mean:100,xsell_max_mean:100000,xsell_min_rows:100000"
SETS="default= xl=xsell:7,$X xlf1=xsell:7,xsell_fold:1,$X xlq23=xsell:7,xsell_q:23,$X xlq14=xsell:7,xsell_q:14,$X xls48=xsell:7,xsell_smem_kb:48,$X xlr128=xsell:7,xsell_rows:128,$X xlA=xsell:1,$X xlG=xsell:6,$X"
t0=$(date +%s)
timeout 3000 python tools/tune_kernels.py --config 5 --solves 1 --out $O/tune_c5_e.json --sets $SETS > $O/tune_c5_e.log 2>&1
echo "tune5: $(( $(date +%s) - t0 )) s" >> $O/steps_e.txt
t0=$(date +%s)
X2="xsell_min_mean:100,xsell_max_mean:100000,xsell_min_rows:30000"
SETS2="default= xl=xsell:7,$X2 xlf1=xsell:7,xsell_fold:1,$X2 xlq23=xsell:7,xsell_q:23,$X2 xls48=xsell:7,xsell_smem_kb:48,$X2"
timeout 900 python tools/tune_kernels.py --config 2 --out $O/tune_c2_e.json --sets $SETS2 > $O/tune_c2_e.log 2>&1
echo "tune2: $(( $(date +%s) - t0 )) s" >> $O/steps_e.txt
