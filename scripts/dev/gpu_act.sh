cd $GRAFT_REPO_ROOT
O=gpurun_out/act
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
for c in 2 1; do for i in 1 2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 >> $O/bench$c.jsonl; done; done
timeout 600 python bench.py --config 5 --K 4096 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench5.json
