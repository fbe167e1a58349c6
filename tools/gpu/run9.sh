mkdir -p gpurun_out
timeout 400 python tools/livelock_probe.py gpu --max-wall 250 > gpurun_out/probe_gpu.log 2>&1
timeout 400 python tools/livelock_probe.py oracle --max-wall 250 > gpurun_out/probe_oracle.log 2>&1
timeout 400 python bench.py --full-run --no-cpu-baseline --verbose --max-wall 200 \
  --dump-ticks gpurun_out/ticks9.json.gz --dump-window 0,400 > gpurun_out/full9.json 2> gpurun_out/full9.err
tail -n 2 gpurun_out/probe_gpu.log gpurun_out/probe_oracle.log
