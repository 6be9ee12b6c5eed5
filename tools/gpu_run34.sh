#!/bin/bash
# W4 slice width 512 (default now) vs 1024: parity + layer timeline + decode step
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_w4_layer.py tests/test_gpu_w4.py -x -q --timeout=300 2>&1 | tail -2
for v in liblarosa liblarosa_w1024 liblarosa liblarosa_w1024; do
  LAROSA_LIB=$PWD/paper_2507_01299_b200/lib/$v.so timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 --w4 > gpurun_out/tlw_$v.json 2>&1
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/tlw_$v.json').read().strip().splitlines()[-1]);print(d['layer_us'], {k:(v.get('loop_max'), v.get('ticket_max'), v.get('exit_max')) for k,v in d['kernels'].items()})")"
done
timeout 600 python tools/w4_decode.py 2>/dev/null | tail -1
