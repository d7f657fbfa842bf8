# plan bench variance / A-B: current build vs HEAD, driving and navigation
cd $GRAFT_REPO_ROOT
O=gpurun_out/ap4
mkdir -p $O
nproc > $O/nproc.txt; lscpu | head -20 >> $O/nproc.txt
for r in 1 2; do
  for v in cur head; do
    if [ $v = cur ]; then unset DESPOT_LIB; else export DESPOT_LIB=$PWD/abtest/libdespot_head.so; fi
    timeout 300 python scripts/plan_bench.py --configs 4 3 --workers 1 8 --no-oracle 2>/dev/null | grep '"gpu"' | sed "s/^/$v /" >> $O/plan_ab.txt
  done
done
