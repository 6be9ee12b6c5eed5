#!/bin/bash
mkdir -p gpurun_out
for f in test_gpu_kernels test_gpu_layer test_gpu_decode test_gpu_modes; do
  timeout 600 python -m pytest tests/$f.py -x -v --timeout=120 > gpurun_out/pt_$f.log 2>&1
  echo "$f rc=$? $(grep -E 'passed|failed|Timeout|timeout' gpurun_out/pt_$f.log | tail -2)"
done
