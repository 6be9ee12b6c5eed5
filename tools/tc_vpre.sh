# tcgen05 GEMV value look-ahead (LAROSA_TC_VPRE chunks) at the default 2-stage x 4-CTA ring.
LIB=paper_2507_01299_b200/lib/liblarosa.so
cp $LIB /tmp/lib_default.so
run() { echo "$1 $(timeout 300 python tools/decode_bench.py --batches 8,16 --ps 0.4,0.0)"; }
{
run v1
for V in 2 3; do cp paper_2507_01299_b200/lib/variants/liblarosa_v$V.so $LIB; run v$V; done
cp /tmp/lib_default.so $LIB
run v1_again
} > gpurun_out/tc_vpre.log 2>&1
