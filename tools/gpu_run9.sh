mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_calib.py -q -k "255" 2>&1 | grep -E "^E " | head -12 > gpurun_out/pytest_calib.log
