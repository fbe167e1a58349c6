mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu19.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu19.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke19.log 2>&1; echo "rc=$?" >> gpurun_out/smoke19.log
timeout 300 python tools/attn_bench.py --out gpurun_out/attn_bench19.json > /dev/null 2>&1
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/bench19.json 2> gpurun_out/bench19.err; echo "rc=$?" >> gpurun_out/bench19.err
tail -n 3 gpurun_out/pytest_gpu19.log
