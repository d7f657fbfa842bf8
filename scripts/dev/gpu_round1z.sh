set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python scripts/exp_c1.py > gpurun_out/exp_c1.log 2>&1
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c$c.log
done
