import sys, torch, json
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.calibration_extra("cuda:0")))
