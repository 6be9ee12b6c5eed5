import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, synth
shape = synth.MODELS["llama2-7b"]
layers = bench.build_stack(shape, "cuda:0", 1)
print(json.dumps(bench.prefill_extra(layers, shape, "cuda:0")))
