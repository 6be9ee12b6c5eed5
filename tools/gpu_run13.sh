mkdir -p gpurun_out
rm -f gpurun_out/b1_sweep.json
run() { env "$@" python tools/b1_layer_us.py >> gpurun_out/b1_sweep.json 2>> gpurun_out/b1_sweep.err; }
run LAROSA_X=0
run LAROSA_COMP_LATE=1
run LAROSA_X=0
run LAROSA_COMP_LATE=1
