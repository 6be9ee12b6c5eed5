#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_w4_layer.py tests/test_gpu_w4.py -x -q --timeout=300 2>&1 | tail -1
for f in 0 512 1024; do
  LAROSA_W4_SLICE=$f timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 --w4 > gpurun_out/tlw_$f.json 2>&1
  echo "slice=$f $(python -c "import json;d=json.loads(open('gpurun_out/tlw_$f.json').read().strip().splitlines()[-1]);print(d['layer_us'], {k:v.get('exit_max') for k,v in d['kernels'].items()})")"
done
timeout 600 python tools/w4_decode.py 2>/dev/null | tail -1
