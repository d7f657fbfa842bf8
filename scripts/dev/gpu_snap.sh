cd $GRAFT_REPO_ROOT
O=gpurun_out/sn
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
for c in 1 2 3; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench$c.json; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_config3.csv python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_config2.csv python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l2.log 2>&1
