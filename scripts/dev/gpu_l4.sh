cd $GRAFT_REPO_ROOT
O=gpurun_out/l4
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_config4.csv python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k3_ -s 6 -c 2 -o $O/k3_config4 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_k3_4.log 2>&1
