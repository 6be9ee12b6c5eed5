#!/bin/bash
# DRAM traffic and launch list of ONE decode step of the bench workload (bench.py --traffic-probe):
# every kernel inside the NVTX range "traffic_step" (one CUDA-graph replay), with its duration and
# dram bytes read + written.  Writes gpurun_out/traffic_B<b>_p<p>.csv; summarise with
# tools/traffic_summarize.py into profiles/traffic.json (keyed by the library source hash).
# Usage (on the GPU box): bash tools/traffic.sh <batch> <p>
set -e
B=${1:-1}; P=${2:-0.4}
mkdir -p gpurun_out
python bench.py --traffic-probe --batch $B --p $P --warmup 3 > gpurun_out/traffic_plain_B${B}.log 2>&1
ncu --nvtx --nvtx-include "traffic_step/" --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --print-units base \
    --csv --log-file gpurun_out/traffic_B${B}_p${P}.csv \
    python bench.py --traffic-probe --batch $B --p $P --warmup 3 > gpurun_out/traffic_ncu_B${B}.log 2>&1
