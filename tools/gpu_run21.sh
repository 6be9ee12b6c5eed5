#!/bin/bash
mkdir -p gpurun_out
for m in 2 3 1; do
  echo "mode=$m $(LAROSA_RULE_KERNEL=$m P=0.4 timeout 300 python tools/b16_phases.py 2>&1 | tail -1)"
done
