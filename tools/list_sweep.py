"""Run bench_extras.list_gemv_sweep_extra alone (JSON)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import bench_extras as BX  # noqa: E402
torch.cuda.set_device(0)
peaks, _ = bench.measured_peaks()
print(json.dumps(BX.list_gemv_sweep_extra("cuda:0", peaks)))
