set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
DESPOT_LIB=$PWD/abtest/libdespot_car128x4.so timeout 300 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_ab.log 2>&1
timeout 300 python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o gpurun_out/prof_k2_c1n python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
