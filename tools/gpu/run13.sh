mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu13.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu13.log
timeout 700 python bench.py --verbose --profile-hooks > gpurun_out/bench13.json 2> gpurun_out/bench13.err; echo "rc=$?" >> gpurun_out/bench13.err
timeout 300 python bench_swap.py --wt-only --out gpurun_out/wt_chunks13.json > gpurun_out/wt_chunks13.log 2>&1
timeout 900 python bench.py --config c4 --steps 200 --verbose --no-cpu-baseline > gpurun_out/c4_13.json 2> gpurun_out/c4_13.err; echo "rc=$?" >> gpurun_out/c4_13.err
tail -n 3 gpurun_out/pytest_gpu13.log
