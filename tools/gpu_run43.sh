#!/bin/bash
# prefill GEMM: TMA multicast clusters (1 / 2 / 4) -- parity then timing, each under a short timeout
for c in 4 2 1; do
  echo "cluster=$c $(LAROSA_PF_CLUSTER=$c timeout 300 python -m pytest tests/test_gpu_prefill.py -x -q --timeout=120 2>&1 | tail -1)"
done
for c in 1 2 4; do
  echo "cluster=$c $(LAROSA_PF_CLUSTER=$c timeout 200 python tools/prefill_time.py 2>&1 | tail -1 | python -c '
import json,sys
d=json.loads(sys.stdin.read())
print({n:(round(v["bf16"]["ms"],4), round(v["cublas_dense_bf16_ms"],4)) for n,v in d.items()})')"
done
