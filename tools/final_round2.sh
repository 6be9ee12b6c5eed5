#!/bin/bash
# Round-2 evidence at the final sources: full GPU suite, smoke, the default bench line, the
# reference arm, the ncu launch list and one ncu --set full capture of the SELECT GEMV sites.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench_rc=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref_rc=$?
python tools/probe_layer.py 0.4 llama3-8b > gpurun_out/plain.log 2>&1; echo probe_rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 8 -c 4 -o gpurun_out/prof_gemv_r02 \
    python tools/probe_layer.py 0.4 llama3-8b > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
