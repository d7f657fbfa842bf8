# round profile refresh, part B: sweeps and the host tree driver
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r01
mkdir -p $O
timeout 1500 python scripts/sweep.py > $O/sweep_config5.jsonl 2>&1
timeout 900 python scripts/peds_sweep.py > $O/peds_sweep.jsonl 2>&1
timeout 900 python scripts/plan_bench.py --configs 1 2 3 4 --workers 1 4 8 > $O/plan_bench.jsonl 2>&1
timeout 1000 python scripts/next2_sweeps.py > $O/next2_sweeps.jsonl 2>&1
timeout 1200 python scripts/online_bench.py --episodes 6 --budgets 0.02 0.1 0.3 --steps 30 > $O/online.jsonl 2>&1
g++ -O2 -std=c++17 scripts/latency.cpp -Iinclude -I/usr/local/cuda/include -Lpaper_1802_06215_b200 -ldespot \
  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1802_06215_b200 -o /tmp/latency && \
  timeout 120 /tmp/latency > $O/latency.jsonl 2>&1
# functional run of the N > 1 bench path on this one GPU (gloo, host-staged): not a measurement
for c in 2 4 1; do
  DESPOT_BENCH_ONE_GPU_TEST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$c bench.py --gpus 2 --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{'
done > $O/bench_n2_functional.jsonl
