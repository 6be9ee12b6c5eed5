mkdir -p gpurun_out
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_decode.py tests/test_gpu_decode_full.py tests/test_gpu_w4.py -q -x 2>&1 | tail -3 > gpurun_out/p.log
rm -f gpurun_out/b1_sweep.json
for i in 1 2; do python tools/b1_layer_us.py >> gpurun_out/b1_sweep.json 2>> gpurun_out/b1_sweep.err; done
python tools/layer_timeline.py --model llama3-8b --p 0.4 > gpurun_out/tl_l3_p04.json 2> gpurun_out/tl.err
