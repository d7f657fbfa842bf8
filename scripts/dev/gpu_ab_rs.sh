# A/B of the RockSample K2 occupancy target (kMinBlocks 8 / 7 / 6), config 2 and 5 (K=4096); parity of the default
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_parity.txt
for v in default rs7 rs6 default; do
  if [ $v = default ]; then unset DESPOT_LIB; else export DESPOT_LIB=$PWD/abtest/libdespot_$v.so; fi
  timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench2_$v.json
  timeout 600 python bench.py --config 5 --K 4096 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench5_$v.json
done
