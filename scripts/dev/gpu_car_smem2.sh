# driving thread kernel with the policy gap fused into step: registers vs shared memory
cd $GRAFT_REPO_ROOT
O=gpurun_out/cs2
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "car or config4 or rollout" > $O/pytest_car.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_car.txt
HD_CAR_SMEM=1 timeout 900 python -m pytest tests -m gpu -q -x -k "car or config4" > $O/pytest_car_smem.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_car_smem.txt
for v in 0 1 0 1; do
  HD_CAR_SMEM=$v timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 >> $O/bench4_smem$v.jsonl
done
