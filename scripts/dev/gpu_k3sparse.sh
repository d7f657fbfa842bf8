cd $GRAFT_REPO_ROOT
O=gpurun_out/ks
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
for i in 1 2; do timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 >> $O/bench4.jsonl; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_config4.csv python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l4.log 2>&1
