#!/bin/bash
for cfg in "0 130" "20 130" "25 130" "40 130" "25 100" "33 100" "25 160"; do
  set -- $cfg
  LAROSA_COMP_PCT=$1 LAROSA_COMP_WAVE_PCT=$2 timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 > gpurun_out/tl_cp.json 2>&1
  echo "pct=$1 wave=$2 $(python -c "import json;d=json.loads(open('gpurun_out/tl_cp.json').read().strip().splitlines()[-1]);k=d['kernels'];print(d['layer_us'], k['down_select']['exit_max'], k['down_companion']['exit_max'], k['down_select']['ctas'], k['down_companion']['ctas'])")"
done
