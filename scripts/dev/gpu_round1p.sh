set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python scripts/plan_bench.py --configs 1 2 3 4 --budget 1.0 > gpurun_out/plan_bench.log 2>&1
