mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
TF_ATTN_IMPL=4 timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x > gpurun_out/pytest_v4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v4.log
TF_ATTN_IMPL=4 timeout 300 python tools/attn_bench.py --out gpurun_out/attn_bench_v4b.json > gpurun_out/attn_bench_v4b.log 2>&1
timeout 900 python bench.py --full-run --no-cpu-baseline --verbose --watchdog 30 --max-wall 700 > gpurun_out/full4.json 2> gpurun_out/full4.err; echo "rc=$?" >> gpurun_out/full4.err
tail -n 3 gpurun_out/pytest_gpu4.log
