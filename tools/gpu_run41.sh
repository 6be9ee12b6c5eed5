#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_layer.py tests/test_gpu_decode.py tests/test_gpu_decode_full.py tests/test_gpu_shard.py tests/test_gpu_modes.py -x -q --timeout=300 2>&1 | tail -1
python tools/b16_timeline.py > gpurun_out/b16tl8.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/b16tl8.json').read().strip().splitlines()[-1])
for k,v in d['kernels'].items():
    if k.startswith('topk'): print(k, v)"
echo "b16 $(P=0.4 timeout 300 python tools/b16_phases.py 2>&1 | tail -1)"
