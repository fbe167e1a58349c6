# ncu captures + C5 sweep (round-1 profiles)
mkdir -p gpurun_out
for impl in 3 4; do
  for case in 64:short736:exact 128:uniform2600:exact; do
    tag=$(echo $case | cut -d: -f1,2 | tr ':' '_')
    TF_ATTN_IMPL=$impl timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn -c 1 \
      -o gpurun_out/attn_v${impl}_${tag} -f python tools/attn_bench.py --only $case --reps 1 --out /tmp/x.json \
      > gpurun_out/ncu_attn_v${impl}_${tag}.log 2>&1
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" -c 3000 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline \
  > gpurun_out/ncu_bench.log 2>&1
timeout 1500 python bench_swap.py --max-blocks 65536 --host-blocks 16384 --engines 0,1 --overlap \
  --out gpurun_out/swap_sweep_64k.json > gpurun_out/swap_sweep.log 2>&1
echo done
