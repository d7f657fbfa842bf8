cd $GRAFT_REPO_ROOT
O=gpurun_out/dc
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
for c in 1 3 2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench$c.json; done
DESPOT_HOST_TRACE=1 timeout 300 python scripts/dev/host_trace.py > $O/host_trace.txt 2>&1
timeout 600 python scripts/plan_bench.py --configs 1 3 --workers 1 8 > $O/plan_bench.jsonl 2>&1
