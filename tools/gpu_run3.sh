mkdir -p gpurun_out
python tools/layer_timeline.py --model llama3-8b --p 0.4 > gpurun_out/tl_l3_p04.json 2> gpurun_out/tl.err
python tools/layer_timeline.py --model llama3-8b --p 0.0 > gpurun_out/tl_l3_p00.json 2>> gpurun_out/tl.err
