cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/profile_iter.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sell|k_csr" -s 35 -c 8 -o gpurun_out/prof_r01b python tools/profile_iter.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
