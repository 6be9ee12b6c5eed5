for pct in 0 35 45 50 55 65; do LAROSA_COMP_PCT=$pct TAG=pct$pct python tools/layer_us.py 0.5 2000; done
ADAPTER=separate TAG=separate python tools/layer_us.py 0.5 2000
