cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/profile_iter.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_iter.py > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?" >> gpurun_out/ncu_list.log
python tools/profile_iter.py > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sell|k_csr|k_sbsr3" -s 43 -c 14 -o gpurun_out/prof_r01 python tools/profile_iter.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
