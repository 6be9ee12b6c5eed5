mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest.log
python tools/layer_timeline.py --model llama3-8b --p 0.4 > gpurun_out/tl_l3_p04.json 2> gpurun_out/tl.err
for m in 1 2 3; do
LAROSA_ATTN=$m python bench.py --steps 50 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/b1_m$m.json 2> gpurun_out/b1.err
LAROSA_ATTN=$m python bench.py --steps 50 --warmup 5 --no-extras --no-cpu-baseline --batch 16 > gpurun_out/b16_m$m.json 2> gpurun_out/b16.err
done
