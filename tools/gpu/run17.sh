mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu17.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu17.log
timeout 700 python bench.py > gpurun_out/bench17.json 2> gpurun_out/bench17.err; echo "rc=$?" >> gpurun_out/bench17.err
timeout 500 python bench.py --full-run --no-cpu-baseline --max-wall 300 > gpurun_out/full17.json 2> gpurun_out/full17.err
tail -n 3 gpurun_out/pytest_gpu17.log
