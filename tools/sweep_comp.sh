TAG=respre python tools/layer_us.py 0.5 3000
TAG=respre2 python tools/layer_us.py 0.5 3000
