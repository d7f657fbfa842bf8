set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
g++ -O2 -std=c++17 scripts/latency.cpp -Iinclude -I/usr/local/cuda/include -Lpaper_1802_06215_b200 -ldespot \
  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1802_06215_b200 -o /tmp/latency
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k3_small -s 3 -c 1 -o gpurun_out/prof_k3small /tmp/latency 20 > gpurun_out/ncu_a.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_a.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k2_expand -s 10 -c 1 -o gpurun_out/prof_k2fused /tmp/latency 20 > gpurun_out/ncu_b.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_b.log
