cd $GRAFT_REPO_ROOT
for c in 2 4 1; do
DESPOT_BENCH_ONE_GPU_TEST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$c bench.py --gpus 2 --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_c$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n2_c$c.log
done
