# driving thread kernel: pedestrians in registers vs in shared memory (HD_CAR_SMEM=1)
cd $GRAFT_REPO_ROOT
O=gpurun_out/cs
mkdir -p $O
HD_CAR_SMEM=1 timeout 900 python -m pytest tests -m gpu -q -x -k "car or config4" > $O/pytest_car_smem.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_car_smem.txt
for v in 0 1 0 1; do
  HD_CAR_SMEM=$v timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 >> $O/bench4_smem$v.jsonl
done
HD_CAR_SMEM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_car -s 3 -c 1 -o $O/k2_car_smem python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu4.log 2>&1
