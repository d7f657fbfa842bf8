set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_search_gpu.py -q -x > gpurun_out/pytest_search.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_search.log
timeout 600 python scripts/plan_bench.py --configs 1 2 3 4 --workers 1 4 8 > gpurun_out/plan.log 2>&1; echo "rc=$?" >> gpurun_out/plan.log
