mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rs -x 2>&1 | tail -12 > gpurun_out/pytest_all.log
