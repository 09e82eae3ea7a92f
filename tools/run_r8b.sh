# C5 full size, call B: the CPU oracle solve on the hierarchy call A cached in /tmp
# (same box, reused within 5 minutes); skipped when the cache is gone.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export ASPAMG_CACHE_DIR=/tmp/aspamg_cache
ls -la /tmp/aspamg_cache > gpurun_out/cache_b.txt 2>&1
if ls /tmp/aspamg_cache/hier_c5_s1_*.bin > /dev/null 2>&1; then
  timeout 2700 python tools/full_configs.py --configs 5 --out gpurun_out/full_configs_c5.json > gpurun_out/full_configs_c5b.log 2>&1
  echo "c5b rc=$?" >> gpurun_out/full_configs_c5b.log
else
  echo "no cached C5 hierarchy on this box" > gpurun_out/full_configs_c5b.log
fi
