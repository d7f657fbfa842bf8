# REDUX-based exact int64 warp sums: parity, configs 1/2/3 bench, ncu source capture of config 2 K2
cd $GRAFT_REPO_ROOT
O=gpurun_out/rx
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
for c in 2 1 3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o $O/k2_config2 python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu2.log 2>&1
