#!/bin/bash
mkdir -p gpurun_out
for h in 4 2 1; do
  echo "hpc=$h $(LAROSA_ATTN_HPC=$h P=0.4 timeout 300 python tools/b16_phases.py 2>&1 | tail -1)"
done
