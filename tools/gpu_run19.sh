#!/bin/bash
# topk kernel writes the batch-16 token image (no rule_apply_image launch): parity + layer times
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_layer.py tests/test_gpu_decode.py tests/test_gpu_decode_full.py tests/test_gpu_modes.py -x -q 2>&1 | tail -5
for ti in 0 1; do
  for p in 0.4 0.0; do
    echo "topk_image=$ti p=$p $(LAROSA_TOPK_IMAGE=$ti P=$p timeout 300 python tools/b16_phases.py 2>&1 | tail -1)"
  done
done
