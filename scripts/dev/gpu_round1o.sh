set -x
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --plan --plan-configs 1 2 --plan-budget 0.3 > gpurun_out/plan_mode.log 2>&1; echo "rc=$?" >> gpurun_out/plan_mode.log
timeout 900 python scripts/online_bench.py --episodes 3 --budgets 0.02 0.1 --steps 20 > gpurun_out/online.jsonl 2> gpurun_out/online.err; echo "rc=$?" >> gpurun_out/online.err
