# A/B of the navigation K2 and driving thread-kernel occupancy targets
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab2
mkdir -p $O
for v in default nav4 nav6; do
  if [ $v = default ]; then unset DESPOT_LIB; else export DESPOT_LIB=$PWD/abtest/libdespot_$v.so; fi
  timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench3_$v.json
done
for v in default cart4 cart5; do
  if [ $v = default ]; then unset DESPOT_LIB; else export DESPOT_LIB=$PWD/abtest/libdespot_$v.so; fi
  timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench4_$v.json
done
