cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "config3 or small_full or mixed or rollout_bounds" > gpurun_out/pytest_nav.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nav.log
timeout 300 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
