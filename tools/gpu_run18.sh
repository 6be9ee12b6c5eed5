#!/bin/bash
# W4 down companion share sweep (layer timeline, LLaMA3-8B p = 0.4)
mkdir -p gpurun_out
for pct in 25 35 45 55; do
  LAROSA_W4_COMP_PCT=$pct timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 --w4 > gpurun_out/tl_w4_c$pct.json 2>&1
  echo pct=$pct $(python -c "import json;d=json.loads(open('gpurun_out/tl_w4_c$pct.json').read().strip().splitlines()[-1]);print(d['layer_us'], d['kernels']['down_select']['exit_max'], d['kernels']['down_companion']['exit_max'])")
done
