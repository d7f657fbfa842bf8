set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c$c.log
done
timeout 600 python scripts/plan_bench.py --configs 1 3 4 --budget 1.0 --no-oracle > gpurun_out/plan_bench.log 2>&1
timeout 300 python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o gpurun_out/prof_k2_c1 python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_group -s 3 -c 1 -o gpurun_out/prof_k3_c4 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1
echo "rc=$?" >> gpurun_out/ncu4.log
