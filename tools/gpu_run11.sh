mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/pytest_all.log
bash tools/traffic.sh 16 0.4; echo "traffic16 rc=$?"
