set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c$c.log
done
timeout 300 python bench.py --config 5 --K 8192 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 6 -c 1 -o gpurun_out/prof_k2_c2e python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 6 -c 1 -o gpurun_out/prof_k2_c4e python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full4.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
