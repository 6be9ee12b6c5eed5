for w in 100 115 130 150; do LAROSA_SEL_WAVE_PCT=$w TAG=selwave$w python tools/layer_us.py 0.5 3000; done
