#!/bin/bash
# prefill GEMM variants: stages / CTAs per SM
mkdir -p gpurun_out
for v in liblarosa liblarosa_pf22 liblarosa_pf31; do
  echo "$v $(LAROSA_LIB=$PWD/paper_2507_01299_b200/lib/$v.so timeout 300 python tools/prefill_time.py 2>&1 | tail -1 | python -c '
import json,sys
d=json.loads(sys.stdin.read())
print({n:(round(v["bf16"]["ms"],4), round(v["cublas_dense_bf16_ms"],4)) for n,v in d.items()})')"
done
timeout 600 env LAROSA_LIB=$PWD/paper_2507_01299_b200/lib/liblarosa_pf22.so python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -2
