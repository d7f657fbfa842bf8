set -x
cd $GRAFT_REPO_ROOT
for mb in 5 6 8; do
  DESPOT_LIB=$PWD/abtest/libdespot_nav$mb.so timeout 300 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/nav_mb$mb.log 2>&1
done
DESPOT_LIB=$PWD/abtest/libdespot_nav5.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "config3 or small_full or mixed" > gpurun_out/pytest_nav.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nav.log
