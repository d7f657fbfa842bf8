# narrow K2 tiles for item-poor batches: tests, configs 1-3 bench, config 3 ncu
cd $GRAFT_REPO_ROOT
O=gpurun_out/tw
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
for c in 1 2 3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o $O/k2_config3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_config3.csv python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l3.log 2>&1
