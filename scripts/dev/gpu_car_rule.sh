cd $GRAFT_REPO_ROOT
O=gpurun_out/cr
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 900 python scripts/peds_sweep.py > $O/peds_sweep.jsonl 2>&1
timeout 600 python scripts/plan_bench.py --configs 4 --workers 1 8 > $O/plan_bench4.jsonl 2>&1
