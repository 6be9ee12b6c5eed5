#!/bin/bash
run() { timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 > gpurun_out/tl_x.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/tl_x.json').read().strip().splitlines()[-1]);print(d['layer_us'])"; }
for v in liblarosa liblarosa_gs3 liblarosa_gs6; do echo "$v $(LAROSA_LIB=$PWD/paper_2507_01299_b200/lib/$v.so run)"; done
for w in 70 85 115 130; do echo "selwave=$w $(LAROSA_SEL_WAVE_PCT=$w run)"; done
for c in 1 2 3; do echo "ctas_per_sm=$c $(LAROSA_GEMV_CTAS_PER_SM=$c run)"; done
