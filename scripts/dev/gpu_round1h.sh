set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c$c.log
done
timeout 300 python bench.py --config 5 --K 32768 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 600 python scripts/plan_bench.py --configs 1 2 3 4 --budget 1.0 > gpurun_out/plan_bench.log 2>&1; echo "plan rc=$?" >> gpurun_out/plan_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 6 -c 1 -o gpurun_out/prof_k2_c2h python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
