set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "car_sharded or sharded_model or fake_ranks" > gpurun_out/pytest_shard.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_shard.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
