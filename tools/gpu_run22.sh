#!/bin/bash
# P2P push path of the sharded decode step: emulation + world-1 symmetric memory
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_shard.py -x -q 2>&1 | tail -15
