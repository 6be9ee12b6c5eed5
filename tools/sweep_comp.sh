TAG=early python tools/layer_us.py 0.5 3000
LAROSA_PDL_LATE=1 TAG=late python tools/layer_us.py 0.5 3000
