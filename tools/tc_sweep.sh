# Batch-8/16 decode step (LLaMA3-8B, 32 layers + head) vs the tcgen05 GEMV grid target
# (LAROSA_TC_TARGET_PCT = CTAs per SM x 100) and vs the CUDA-core batched GEMV (LAROSA_GEMV_TC=0).
for t in 100 150 200 300; do
  echo "target_pct=$t $(LAROSA_TC_TARGET_PCT=$t timeout 300 python tools/decode_bench.py --batches 8,16 --ps 0.4,0.0)"
done
echo "cuda_core $(LAROSA_GEMV_TC=0 timeout 300 python tools/decode_bench.py --batches 8,16 --ps 0.4,0.0)"
