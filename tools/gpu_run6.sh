mkdir -p gpurun_out
python -m pytest tests/test_gpu_shard.py -x -q -rs 2>&1 | tail -15 > gpurun_out/pytest_shard.log
