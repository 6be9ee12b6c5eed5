#!/bin/bash
# W4A16 layer integration: parity + the W4 decode-step timing
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_w4_layer.py tests/test_gpu_w4.py tests/test_abi_cpu.py -x -q 2>&1 | tail -30
timeout 600 python tools/w4_decode.py > gpurun_out/w4_decode.json 2> gpurun_out/w4_decode.err; echo rc=$?
cat gpurun_out/w4_decode.json; tail -5 gpurun_out/w4_decode.err
