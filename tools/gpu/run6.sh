mkdir -p gpurun_out
timeout 600 python bench.py --verbose > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "rc=$?" >> gpurun_out/bench6.err
timeout 900 python bench.py --full-run --no-cpu-baseline --verbose --watchdog 30 --max-wall 700 > gpurun_out/full6.json 2> gpurun_out/full6.err; echo "rc=$?" >> gpurun_out/full6.err
bash tools/gpu/run5.sh
