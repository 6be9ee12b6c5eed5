set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q -rs -s -k "p0_equals or residual_adapter or p5 or graph_replay or decode or extreme" 2>&1 | grep -v "^$" | tail -40 > gpurun_out/pytest_a.log
python -m pytest tests -m gpu -q -rs 2>&1 | tail -15 > gpurun_out/pytest_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
