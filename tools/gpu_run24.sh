#!/bin/bash
mkdir -p gpurun_out
for v in liblarosa liblarosa_nf; do
  for c in p2p nccl; do
    LAROSA_LIB=$PWD/paper_2507_01299_b200/lib/$v.so timeout 900 python bench.py --workload sharded-70b --collective $c --batch 1 --layers 20 --steps 20 --warmup 3 > gpurun_out/sh_${v}_${c}.json 2>&1
    echo "$v $c $(python -c "import json;d=json.loads(open('gpurun_out/sh_${v}_${c}.json').read().strip().splitlines()[-1]);print(d['ms_per_step'])")"
  done
done
