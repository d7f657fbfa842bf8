cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "car" > gpurun_out/pytest_car.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_car.log
for mb in 1 5 6 8; do
  DESPOT_LIB=$PWD/abtest/libdespot_cg$mb.so timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --car-variant group > gpurun_out/carg_mb$mb.log 2>&1
done
for v in thread warp; do timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --car-variant $v > gpurun_out/carg_$v.log 2>&1; done
for peds in 6 12; do for v in thread group; do timeout 300 python bench.py --config 4 --peds $peds --steps 10 --warmup 3 --no-cpu-baseline --car-variant $v > gpurun_out/carg_p${peds}_$v.log 2>&1; done; done
for v in thread group warp; do timeout 300 python bench.py --config 4 --K 64 --steps 10 --warmup 3 --no-cpu-baseline --car-variant $v > gpurun_out/carg_k64_$v.log 2>&1; done
