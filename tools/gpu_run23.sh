#!/bin/bash
# sharded LLaMA3-70B step at n = 1: NCCL all-gather vs P2P push (symmetric memory)
mkdir -p gpurun_out
for c in nccl p2p; do
  for b in 1 16; do
    timeout 900 python bench.py --workload sharded-70b --collective $c --batch $b --steps 10 --warmup 3 > gpurun_out/sh70_${c}_b$b.json 2> gpurun_out/sh70_${c}_b$b.err
    echo "$c B=$b rc=$? $(tail -c 400 gpurun_out/sh70_${c}_b$b.json | head -c 300)"
  done
done
