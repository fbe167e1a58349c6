# is the small-batch attention time set by address translation / page locality?  (tag = $1)
T=${1:-r2tlb}
mkdir -p gpurun_out
for lay in random contig; do
  for pb in 22000 6000; do
    echo "== layout $lay pool $pb" >> gpurun_out/${T}.log
    timeout 300 python tools/attn_bench.py --impls 3,5 --plans pool --batches 32,128 --layout $lay --pool-blocks $pb --out gpurun_out/${T}_${lay}_${pb}.json 2>&1 | grep -v uniform >> gpurun_out/${T}.log
  done
done
cat gpurun_out/${T}.log
