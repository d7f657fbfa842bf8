# lane-refill K2: parity, config 3 both forms, ncu of the refill kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/rf
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_parity.txt
for f in tiles refill; do
  timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline --k2-form $f > $O/bench3_$f.log 2>&1
done
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --k2-form refill > $O/bench2_refill.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o $O/k2_config3_refill python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu3.log 2>&1
