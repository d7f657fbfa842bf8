set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l3.log 2>&1
