set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c$c.log
done
timeout 300 python bench.py --config 5 --K 4096 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
timeout 600 ncu --metrics smsp__thread_inst_executed.sum,smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:k2_ -c 4 --csv --log-file gpurun_out/k2m.csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k2m.log 2>&1
