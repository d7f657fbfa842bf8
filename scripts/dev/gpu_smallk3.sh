cd $GRAFT_REPO_ROOT
for v in 4096 128; do
  echo "DESPOT_SMALL_K3_MAX=$v" >> gpurun_out/smallk3.log
  DESPOT_SMALL_K3_MAX=$v DESPOT_SEARCH_TRACE=1 python scripts/exp_plan.py 2 >> gpurun_out/smallk3.log 2>&1
  DESPOT_SMALL_K3_MAX=$v DESPOT_SEARCH_TRACE=1 python scripts/exp_plan.py 1 >> gpurun_out/smallk3.log 2>&1
done
