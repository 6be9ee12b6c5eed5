TAG=s4 python tools/layer_us.py 0.5 3000
LAROSA_LIB=$PWD/paper_2507_01299_b200/lib/liblarosa_s3.so TAG=s3 python tools/layer_us.py 0.5 3000
LAROSA_LIB=$PWD/paper_2507_01299_b200/lib/liblarosa_s6.so TAG=s6 python tools/layer_us.py 0.5 3000
