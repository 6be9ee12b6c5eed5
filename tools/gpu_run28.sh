#!/bin/bash
mkdir -p gpurun_out
python tools/b16_phases.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rule_select -s 4 -c 2 -o gpurun_out/prof_rule \
    python bench.py --traffic-probe --batch 16 --p 0.4 --warmup 3 > gpurun_out/ncu_rule.log 2>&1; echo full_rc=$?
