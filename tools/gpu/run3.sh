mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
timeout 300 python tools/attn_bench.py --out gpurun_out/attn_bench_v4.json > gpurun_out/attn_bench_v4.log 2>&1
TF_ATTN_IMPL=3 timeout 300 python tools/attn_bench.py --out gpurun_out/attn_bench_v3.json > gpurun_out/attn_bench_v3.log 2>&1
timeout 600 python bench.py --verbose > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "rc=$?" >> gpurun_out/bench3.err
timeout 900 python bench.py --full-run --no-cpu-baseline --verbose --watchdog 20 > gpurun_out/full3.json 2> gpurun_out/full3.err; echo "rc=$?" >> gpurun_out/full3.err
tail -n 3 gpurun_out/pytest_gpu3.log
