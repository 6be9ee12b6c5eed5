TAG=prefetch python tools/layer_us.py 0.5 3000
LAROSA_ADAPTER_PREFETCH=0 TAG=noprefetch python tools/layer_us.py 0.5 3000
