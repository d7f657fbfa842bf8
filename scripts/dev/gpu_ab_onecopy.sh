# A/B: small-batch setup in one host->device copy (current tree) vs HEAD
cd $GRAFT_REPO_ROOT
O=gpurun_out/oc
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for r in 1 2; do for v in cur head; do
  if [ $v = cur ]; then unset DESPOT_LIB; else export DESPOT_LIB=$PWD/abtest/libdespot_head.so; fi
  timeout 600 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/$v /" >> $O/bench1.txt
  timeout 300 python scripts/plan_bench.py --configs 1 --workers 1 8 --no-oracle 2>/dev/null | grep '"gpu"' | sed "s/^/$v /" >> $O/plan1.txt
done; done
