#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_layer.py tests/test_gpu_decode.py tests/test_gpu_modes.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
python tools/b16_timeline.py > gpurun_out/b16tl7.json 2>&1
echo "b16 $(P=0.4 timeout 300 python tools/b16_phases.py 2>&1 | tail -1)"
timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 > gpurun_out/tl_attn.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/tl_attn.json').read().strip().splitlines()[-1]);print('b1', d['layer_us'], d['kernels']['attention'])"
