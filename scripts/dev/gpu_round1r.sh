set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
g++ -O2 -std=c++17 scripts/latency.cpp -Iinclude -I/usr/local/cuda/include -Lpaper_1802_06215_b200 -ldespot \
  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1802_06215_b200 -o /tmp/latency && \
  timeout 120 /tmp/latency > gpurun_out/latency.log 2>&1; echo "latency rc=$?" >> gpurun_out/latency.log
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c$c.log
done
