# ncu launch list + one --set full capture of 8 SpMV-family launches of the profiled iteration.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/profile_iter.py > gpurun_out/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_iter.py > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?" >> gpurun_out/ncu_list.log
SKIP=$(grep -cE "^(smooth|resid|restrict|prolong|pcg_Kp|coarse_|tail_dense)" gpurun_out/plain.log)
echo "skip=$SKIP" > gpurun_out/ncu_skip.txt
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_sbsr3|k_csr|k_sell" -s $SKIP -c 8 -o gpurun_out/prof_full python tools/profile_iter.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
