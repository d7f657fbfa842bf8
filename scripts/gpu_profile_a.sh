# round profile refresh, part A: tests, ncu captures of K2 (raw pages first, so
# the bench lines read this build's traffic and per-pipe figures), per-unit
# figures, bench lines, launch list
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r01
mkdir -p $O profiles/r01
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
for c in 1 2 3 4 5; do
  X=""; [ $c = 5 ] && X="--K 32768"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o $O/k2_config$c python bench.py --config $c $X --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_$c.log 2>&1
  echo "rc=$?" >> $O/ncu_full_$c.log
  ncu -i $O/k2_config$c.ncu-rep --page raw --csv > $O/k2_config${c}_raw.csv 2>/dev/null && cp $O/k2_config${c}_raw.csv profiles/r01/
  [ $c = 2 ] || rm -f $O/k2_config$c.ncu-rep   # gpurun brings back <= 64 MiB: keep config 2's report only
done
timeout 1800 python scripts/measure_istep.py --out $O/i_step.json > $O/i_step.log 2>&1
cp $O/i_step.json profiles/r01/i_step.json
timeout 900 python bench.py > $O/bench_default.log 2>&1   # the driver's default command
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --cpu-budget 10 > $O/bench_config$c.log 2>&1
done
timeout 900 python bench.py --config 5 --K 32768 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_config5.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
# launch list of the default command (cold cache, serialised: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo "rc=$?" >> $O/ncu_launch.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config3.csv python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch3.log 2>&1
