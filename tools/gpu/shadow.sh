mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --dump-ticks gpurun_out/ticks_final.json.gz --dump-window 0,1000 > gpurun_out/bench_shadow.json 2> gpurun_out/bench_shadow.err
echo done
