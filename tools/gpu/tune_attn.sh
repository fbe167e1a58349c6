mkdir -p gpurun_out
for w in 2 3 4 6 8; do for m in 4 8 16; do
  TF_ATTN_IMPL=3 TF_ATTN_WAVES=$w TF_ATTN_MINBLK=$m timeout 120 python tools/attn_bench.py --batches 64,128 --plans exact \
    --reps 10 --out gpurun_out/tune_w${w}_m${m}.json > /dev/null 2>&1
done; done
echo tuned
