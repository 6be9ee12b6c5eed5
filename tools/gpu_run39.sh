#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_layer.py tests/test_gpu_decode.py tests/test_gpu_decode_full.py tests/test_gpu_kernels.py tests/test_gpu_w4.py tests/test_gpu_w4_layer.py -x -q --timeout=300 2>&1 | tail -1
for i in 1 2; do
  timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 > gpurun_out/tl_df.json 2>&1
  echo "df $(python -c "import json;d=json.loads(open('gpurun_out/tl_df.json').read().strip().splitlines()[-1]);print(d['layer_us'], {k:(v.get('rule_pool_med'), v.get('sel_mask_med'), v.get('list_med'), v.get('prologue_med')) for k,v in d['kernels'].items() if 'lookup_data_med' in v})")"
done
