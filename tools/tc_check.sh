# Full GPU parity suite plus the batch-8/16 decode step (tcgen05 GEMV) timing.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
tail -3 gpurun_out/pytest_gpu2.log
{ for t in 400 500; do echo "t$t $(LAROSA_TC_TARGET_PCT=$t timeout 300 python tools/decode_bench.py --batches 1,8,16 --ps 0.4,0.0)"; done; } > gpurun_out/tc_after.log 2>&1
cut -c1-900 gpurun_out/tc_after.log
