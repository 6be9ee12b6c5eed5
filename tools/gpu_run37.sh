#!/bin/bash
for v in liblarosa_ca liblarosa liblarosa_ca liblarosa; do
  LAROSA_LIB=$PWD/paper_2507_01299_b200/lib/$v.so timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 > gpurun_out/tl_$v.json 2>&1
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/tl_$v.json').read().strip().splitlines()[-1]);print(d['layer_us'], {k:(v.get('lookup_data_med'), v.get('rule_coarse_med'), v.get('prologue_med')) for k,v in d['kernels'].items() if 'lookup_data_med' in v})")"
done
