"""Time the W4A16 decode-step extra alone (bench.w4_decode_extra) and print its JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402

if __name__ == "__main__":
    torch.cuda.set_device(0)
    peaks, _ = bench.measured_peaks()
    print(json.dumps(bench.w4_decode_extra(synth.MODELS[bench.MODEL], "cuda:0", peaks)))
