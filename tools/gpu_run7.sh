mkdir -p gpurun_out
python -m pytest tests/test_gpu_shard.py tests/test_gpu_shard_gloo.py -x -q -rs 2>&1 | tail -8 > gpurun_out/pytest_shard.log
timeout 900 python bench.py --workload sharded-70b --steps 10 --warmup 3 > gpurun_out/sh70_b1.json 2> gpurun_out/sh70_b1.err
timeout 900 python bench.py --workload sharded-70b --steps 10 --warmup 3 --batch 16 > gpurun_out/sh70_b16.json 2> gpurun_out/sh70_b16.err
timeout 900 python bench.py --workload sharded-70b --model qwen2.5-72b --steps 10 --warmup 3 > gpurun_out/shq72_b1.json 2> gpurun_out/shq72_b1.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/pytest_shard.log
