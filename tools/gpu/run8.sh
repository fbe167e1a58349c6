mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu8.log
timeout 600 python bench.py --verbose > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo "rc=$?" >> gpurun_out/bench8.err
timeout 300 python bench_swap.py --wt-only --out gpurun_out/wt_chunks.json > gpurun_out/wt_chunks.log 2>&1
timeout 800 python bench.py --arrivals poisson --full-run --no-cpu-baseline --verbose --watchdog 60 --max-wall 600 \
  > gpurun_out/full8p.json 2> gpurun_out/full8p.err; echo "rc=$?" >> gpurun_out/full8p.err
tail -n 3 gpurun_out/pytest_gpu8.log
