TAG=auto python tools/layer_us.py 0.5 3000
LAROSA_ATTN_CHUNK=16 TAG=ch16 python tools/layer_us.py 0.5 3000
LAROSA_ATTN_CHUNK=64 TAG=ch64 python tools/layer_us.py 0.5 3000
