#!/bin/bash
# W4 kernel v2 (16 + q codes, b table, wide epilogue): parity + timeline + decode-step timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_w4_layer.py tests/test_gpu_w4.py -x -q 2>&1 | tail -15
timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 --w4 > gpurun_out/tl_w4.json 2>&1; echo rc=$?
timeout 600 python tools/w4_decode.py > gpurun_out/w4_decode.json 2> gpurun_out/w4_decode.err; echo rc=$?
cat gpurun_out/w4_decode.json
