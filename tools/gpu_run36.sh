#!/bin/bash
for v in liblarosa liblarosa_is5 liblarosa_is6 liblarosa_is8; do
  for p in 0.4 0.0; do
    echo "$v p=$p $(LAROSA_LIB=$PWD/paper_2507_01299_b200/lib/$v.so P=$p timeout 300 python tools/b16_phases.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["layer_us"], d["gemvs_only_us"])')"
  done
done
