TAG=persm2 python tools/layer_us.py 0.5 3000
LAROSA_GEMV_CTAS_PER_SM=1 TAG=persm1 python tools/layer_us.py 0.5 3000
