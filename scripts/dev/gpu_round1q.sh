set -x
cd $GRAFT_REPO_ROOT
g++ -O2 -std=c++17 scripts/latency.cpp -Iinclude -I/usr/local/cuda/include -Lpaper_1802_06215_b200 -ldespot -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1802_06215_b200 -o /tmp/latency && timeout 120 /tmp/latency 3000 > gpurun_out/latency.log 2>&1
echo "rc=$?" >> gpurun_out/latency.log
