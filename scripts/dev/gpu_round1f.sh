set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c$c.log
done
for v in warp thread auto; do
  timeout 300 python bench.py --config 4 --car-variant $v --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_$v.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4_$v.log
done
