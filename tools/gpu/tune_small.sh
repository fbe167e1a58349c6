mkdir -p gpurun_out
for w in 2 3 4 6 8; do TF_ATTN_WAVES=$w timeout 120 python tools/attn_bench.py --batches 16,32,48 --plans exact,pool --reps 10 --out gpurun_out/tsmall_w$w.json > /dev/null 2>&1; done
echo done
