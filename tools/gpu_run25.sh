#!/bin/bash
mkdir -p gpurun_out
for c in 0 1; do
  LAROSA_GEMV_CLUSTER=$c timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 > gpurun_out/tl_cl$c.json 2>&1
  echo "cluster=$c $(python -c "import json;d=json.loads(open('gpurun_out/tl_cl$c.json').read().strip().splitlines()[-1]);print(d['layer_us'], {k:v.get('exit_max') for k,v in d['kernels'].items()})")"
done
