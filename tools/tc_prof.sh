# Batch-16 decode (LLaMA3-8B, 2 layers + head, p = 0.4): ncu launch list of the library's kernels,
# then one ncu --set full capture of the tcgen05 GEMV launches of one layer.
python tools/decode_bench.py --layers 2 --batches 16 --ps 0.4 --reps 3 > gpurun_out/tc_plain.log 2>&1; echo plain_rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv \
    -k "regex:gemv|topk|attention|embed|rms_rows|argmax|union|select_prep" \
    --log-file gpurun_out/tc_launches.csv python tools/decode_bench.py --layers 2 --batches 16 --ps 0.4 --reps 3 > gpurun_out/tc_ncu_list.log 2>&1; echo list_rc=$?
[ "$1" = "full" ] && { ncu --set full --clock-control none --import-source on -k regex:gemv_tc_kernel -s 20 -c 5 -o gpurun_out/prof_tc \
    python tools/decode_bench.py --layers 2 --batches 16 --ps 0.4 --reps 3 > gpurun_out/tc_ncu_full.log 2>&1; echo full_rc=$?; }
true
