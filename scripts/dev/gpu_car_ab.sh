set -x
cd $GRAFT_REPO_ROOT
for mb in 3 4 5 6; do
  DESPOT_LIB=$PWD/abtest/libdespot_mb$mb.so timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/car_mb$mb.log 2>&1
  DESPOT_LIB=$PWD/abtest/libdespot_mb$mb.so timeout 300 python bench.py --config 4 --K 64 --steps 10 --warmup 3 --no-cpu-baseline --car-variant thread > gpurun_out/car_mb${mb}_k64.log 2>&1
done
DESPOT_LIB=$PWD/abtest/libdespot_mb4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "car" > gpurun_out/pytest_car.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_car.log
