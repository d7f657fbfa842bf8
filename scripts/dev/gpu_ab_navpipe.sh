# A/B: navigation roll-out drawing the next step's stream words ahead (current tree) vs HEAD
cd $GRAFT_REPO_ROOT
O=gpurun_out/np
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for r in 1 2; do for v in cur head; do
  if [ $v = cur ]; then unset DESPOT_LIB; else export DESPOT_LIB=$PWD/abtest/libdespot_head.so; fi
  timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/$v /" >> $O/bench3.txt
done; done
