cd $GRAFT_REPO_ROOT
O=gpurun_out/cf
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
for c in 3 4 2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench$c.json
done
