mkdir -p gpurun_out
python -m pytest tests/test_gpu_prefill.py -q -rA 2>&1 | grep -E "^(FAILED)|passed|failed" | head -30 > gpurun_out/pytest_prefill.log
python tools/prefill_time.py > gpurun_out/prefill_time.json 2> gpurun_out/prefill_time.err && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum --clock-control none -k regex:prefill -c 8 --csv --print-units base --log-file gpurun_out/prefill_ncu.csv python tools/prefill_time.py > gpurun_out/prefill_ncu.log 2>&1
