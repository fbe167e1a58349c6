mkdir -p gpurun_out
timeout 900 python bench.py --full-run --no-cpu-baseline --verbose --watchdog 20 > gpurun_out/full2.json 2> gpurun_out/full2.err; echo "rc=$?" >> gpurun_out/full2.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 600 python bench.py --no-cpu-baseline --verbose > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "rc=$?" >> gpurun_out/bench2.err
timeout 900 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu-baseline --verbose > gpurun_out/c4.json 2> gpurun_out/c4.err; echo "rc=$?" >> gpurun_out/c4.err
tail -n 3 gpurun_out/pytest_gpu2.log
