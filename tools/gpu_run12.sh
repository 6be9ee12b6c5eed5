mkdir -p gpurun_out
rm -f gpurun_out/b16_phases.json gpurun_out/b16_bench.json
LAROSA_RULE_KERNEL=3 python -m pytest tests/test_gpu_layer.py tests/test_gpu_decode.py tests/test_gpu_decode_full.py -q -x 2>&1 | tail -2 > gpurun_out/pytest_sub.log
for rk in 2 3; do LAROSA_RULE_KERNEL=$rk python tools/b16_phases.py >> gpurun_out/b16_phases.json 2>> gpurun_out/b16_phases.err; done
for rk in 2 3; do LAROSA_RULE_KERNEL=$rk python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline --batch 16 >> gpurun_out/b16_bench.json 2>> gpurun_out/b16_phases.err; done
