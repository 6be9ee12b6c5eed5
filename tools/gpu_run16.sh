#!/bin/bash
# W4 vs bf16 per-kernel timeline (LLaMA3-8B layer, p = 0.4, separate adapter)
mkdir -p gpurun_out
timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 --adapter separate > gpurun_out/tl_bf16.json 2>&1; echo rc=$?
timeout 300 python tools/layer_timeline.py --model llama3-8b --p 0.4 --w4 > gpurun_out/tl_w4.json 2>&1; echo rc=$?
