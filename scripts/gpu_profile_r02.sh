# round-2 profile refresh (one B200): tests, self-check stress, ncu captures of
# K2 (raw pages first, so that the bench lines read this build's traffic and
# per-pipe figures), per-unit instruction counts, bench lines of every config,
# the reference arm, launch lists, C latency, the config-5 K sweep, the
# pedestrian study, the host tree driver, the functional N = 2 run
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02
mkdir -p $O profiles/r02
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
DESPOT_LIB=$PWD/paper_1802_06215_b200/libdespot_checked.so timeout 900 python scripts/sanitize_cases.py --stress 10 > $O/selfcheck_stress.txt 2>&1; echo "rc=$?" >> $O/selfcheck_stress.txt
for c in 1 2 3 4 5; do
  X=""; [ $c = 5 ] && X="--K 32768"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o $O/k2_config$c python bench.py --config $c $X --steps 1 --warmup 3 --no-cpu-baseline --no-all-cores-baseline > $O/ncu_full_$c.log 2>&1
  echo "rc=$?" >> $O/ncu_full_$c.log
  ncu -i $O/k2_config$c.ncu-rep --page raw --csv > $O/k2_config${c}_raw.csv 2>/dev/null && cp $O/k2_config${c}_raw.csv profiles/r02/
  [ $c = 2 ] || rm -f $O/k2_config$c.ncu-rep   # gpurun brings back <= 64 MiB: keep config 2's report only
done
timeout 1800 python scripts/measure_istep.py --out $O/i_step.json > $O/i_step.log 2>&1
cp $O/i_step.json profiles/r02/i_step.json
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err   # the driver's default command
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --cpu-budget 10 > $O/bench_config$c.json 2> $O/bench_config$c.err
done
timeout 900 python bench.py --config 5 --K 32768 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_config5.json 2> $O/bench_config5.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
# launch lists of the default command and of config 3 (cold cache, serialised: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-all-cores-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config3.csv python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-all-cores-baseline > $O/ncu_launch3.log 2>&1
g++ -O2 -std=c++17 scripts/latency.cpp -Iinclude -I/usr/local/cuda/include -Lpaper_1802_06215_b200 -ldespot \
  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1802_06215_b200 -o /tmp/latency && \
  timeout 120 /tmp/latency 3000 > $O/latency.jsonl 2>&1
timeout 1500 python scripts/sweep.py > $O/sweep_config5.jsonl 2>&1
timeout 900 python scripts/peds_sweep.py > $O/peds_sweep.jsonl 2>&1
timeout 900 python scripts/plan_bench.py --configs 1 2 3 4 --workers 1 4 8 > $O/plan_bench.jsonl 2>&1
# functional run of the N > 1 bench path on this one GPU (gloo, host-staged): not a measurement
for c in 2 4 1; do
  DESPOT_BENCH_ONE_GPU_TEST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$c bench.py --gpus 2 --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{'
done > $O/bench_n2_functional.jsonl
ls -la $O
