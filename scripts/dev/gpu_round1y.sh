set -x
cd $GRAFT_REPO_ROOT
for c in 1 3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c$c.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l3.log 2>&1
