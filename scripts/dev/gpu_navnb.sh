cd $GRAFT_REPO_ROOT
O=gpurun_out/nb
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
for i in 1 2; do timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 >> $O/bench3.jsonl; done
