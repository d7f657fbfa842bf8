set -x
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 6 -c 1 -o gpurun_out/prof_k2_c3i python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
timeout 300 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 6 -c 1 -o gpurun_out/prof_k2_c4i python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1
echo "rc=$?" >> gpurun_out/ncu4.log
