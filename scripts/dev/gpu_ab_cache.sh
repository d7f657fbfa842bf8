# A/B: device scratch cache vs cudaMallocAsync per batch, host tree driver on navigation and MARS
cd $GRAFT_REPO_ROOT
O=gpurun_out/abc
mkdir -p $O
for r in 1 2 3; do
  for v in cache nocache; do
    if [ $v = cache ]; then unset DESPOT_LIB; else export DESPOT_LIB=$PWD/abtest/libdespot_nocache.so; fi
    timeout 300 python scripts/plan_bench.py --configs 3 2 --workers 8 2>/dev/null | grep '"gpu"' | sed "s/^/$v /" >> $O/plan_ab.txt
  done
done
