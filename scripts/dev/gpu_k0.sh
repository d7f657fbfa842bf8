# K0 Philox ceiling: test, default bench, ncu of K0
cd $GRAFT_REPO_ROOT
O=gpurun_out/k0
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "k0 or stream_words" > $O/pytest_k0.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_k0.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench2.log 2>&1
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench4.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k0_ -s 1 -c 1 -o $O/k0 python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_k0.log 2>&1
