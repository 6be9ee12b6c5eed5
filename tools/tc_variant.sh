# A/B of the default library against prebuilt variants lib/variants/liblarosa_<tag>.so on the
# batch-8/16 decode step.   bash tools/tc_variant.sh <tag> [...]
LIB=paper_2507_01299_b200/lib/liblarosa.so
cp $LIB /tmp/lib_default.so
run() { echo "$1 $(timeout 300 python tools/decode_bench.py --batches 8,16 --ps 0.4,0.0)"; }
{
run default
for t in "$@"; do cp paper_2507_01299_b200/lib/variants/liblarosa_$t.so $LIB; run $t; done
cp /tmp/lib_default.so $LIB
run default_again
} > gpurun_out/tc_variant.log 2>&1
