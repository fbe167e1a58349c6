mkdir -p gpurun_out
timeout 400 python bench.py --full-run --no-cpu-baseline --verbose --watchdog 30 --max-wall 200 \
  --dump-ticks gpurun_out/ticks7.json.gz --dump-window 60,150 > gpurun_out/full7.json 2> gpurun_out/full7.err
bash tools/gpu/tune_attn.sh
timeout 1500 python bench_swap.py --max-blocks 65536 --host-blocks 16384 --engines 0,1 --overlap \
  --out gpurun_out/swap_sweep_64k.json > gpurun_out/swap_sweep.log 2>&1
echo done
