# Focused ncu captures of the level-0 smoother kernels of the second profiled
# iteration (G: first k_sell launch of the iteration, G': first k_csr launch).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/profile_iter.py > gpurun_out/plain_g.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sell -s 4 -c 1 -o gpurun_out/prof_g python tools/profile_iter.py > gpurun_out/ncu_g.log 2>&1
echo "g rc=$?" >> gpurun_out/ncu_g.log
ncu --set full --clock-control none --import-source on -k regex:k_csr -s 36 -c 1 -o gpurun_out/prof_gt python tools/profile_iter.py > gpurun_out/ncu_gt.log 2>&1
echo "gt rc=$?" >> gpurun_out/ncu_gt.log
