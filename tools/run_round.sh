# One GPU session: tests, smoke, bench (both arms), then ncu captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
python tools/profile_iter.py > gpurun_out/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_iter.py > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?" >> gpurun_out/ncu_list.log
python tools/profile_iter.py > gpurun_out/plain2.log 2>&1
# skip the warm-up iteration's SpMV-family launches (one per SpMV op line of the op table)
SKIP=$(grep -cE "^(smooth|resid|restrict|prolong|pcg_Kp|coarse_|tail_dense)" gpurun_out/plain2.log)
echo "skip=$SKIP" > gpurun_out/ncu_skip.txt
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_sbsr3|k_csr|k_sell" -s $SKIP -c 8 -o gpurun_out/prof_full python tools/profile_iter.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
