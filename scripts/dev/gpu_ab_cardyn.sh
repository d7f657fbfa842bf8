# A/B: driving thread kernel with per-warp dynamic item chunks (current tree) vs HEAD
cd $GRAFT_REPO_ROOT
O=gpurun_out/cd
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "car or config4 or dist or search" > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for r in 1 2; do for v in cur head; do
  if [ $v = cur ]; then unset DESPOT_LIB; else export DESPOT_LIB=$PWD/abtest/libdespot_head.so; fi
  timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/$v /" >> $O/bench4.txt
done; done
timeout 900 python scripts/peds_sweep.py > $O/peds_sweep.jsonl 2>&1
