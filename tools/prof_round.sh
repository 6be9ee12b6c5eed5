# One GPU call: parity tests, the default bench line, the ncu launch list of chained layer
# steps and one ncu --set full capture of the 4 GEMV launches of a step.  Outputs under gpurun_out/.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python tools/probe_layer.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:gemv_kernel|attention_kernel|select_prep|fold_tc" -c 400 --csv \
    --log-file gpurun_out/launches.csv python tools/probe_layer.py > gpurun_out/ncu_list.log 2>&1; echo list_rc=$?
ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 8 -c 4 -o gpurun_out/prof_gemv \
    python tools/probe_layer.py > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
python tools/layer_timeline.py > gpurun_out/timeline.json 2> gpurun_out/timeline.err; echo tl_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref_rc=$?; cat gpurun_out/ref.json
