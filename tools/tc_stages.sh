# tcgen05 GEMV ring depth x CTAs per SM: the batch-8/16 decode step for the default build and
# prebuilt variants (lib/variants/liblarosa_sS.so, -DLAROSA_TC_STAGES=S) at several grid targets.
LIB=paper_2507_01299_b200/lib/liblarosa.so
cp $LIB /tmp/lib_default.so
run() { echo "$1 $(LAROSA_TC_TARGET_PCT=$2 timeout 300 python tools/decode_bench.py --batches 8,16 --ps 0.4,0.0)"; }
{
run s4_t200 200
for v in "3 300" "3 200" "2 400" "2 300"; do set -- $v; cp paper_2507_01299_b200/lib/variants/liblarosa_s$1.so $LIB; run s$1_t$2 $2; done
cp /tmp/lib_default.so $LIB
run s4_t200_again 200
} > gpurun_out/tc_stages2.log 2>&1
cut -c1-300 gpurun_out/tc_stages2.log
