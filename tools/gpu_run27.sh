#!/bin/bash
# one-CTA rule kernel at batch > 1: parity (layer / decode / shard / modes) + batch-16 timeline + phases
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_layer.py tests/test_gpu_decode.py tests/test_gpu_decode_full.py tests/test_gpu_shard.py tests/test_gpu_modes.py -x -q 2>&1 | tail -3 > gpurun_out/pt27.log; cat gpurun_out/pt27.log
python tools/b16_timeline.py > gpurun_out/b16tl3.json 2>&1
for rc in 1 0; do
  for p in 0.4 0.0; do
    echo "rule_cta=$rc p=$p $(LAROSA_RULE_CTA=$rc P=$p timeout 300 python tools/b16_phases.py 2>&1 | tail -1)"
  done
done
