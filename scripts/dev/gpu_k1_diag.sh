# K1 / K3 / host-overhead diagnostics on configs 2 and 3
cd $GRAFT_REPO_ROOT
O=gpurun_out/k1
mkdir -p $O
for c in 2 3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_update -s 3 -c 1 -o $O/k1_config$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_k1_$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_ -s 9 -c 3 -o $O/k3_config3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_k3_3.log 2>&1
DESPOT_HOST_TRACE=1 timeout 300 python scripts/dev/host_trace.py > $O/host_trace.txt 2>&1
