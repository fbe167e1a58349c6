mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu12.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu12.log
timeout 700 python bench.py --verbose > gpurun_out/bench12.json 2> gpurun_out/bench12.err; echo "rc=$?" >> gpurun_out/bench12.err
timeout 900 python bench.py --config c4 --verbose --no-cpu-baseline > gpurun_out/c4_12.json 2> gpurun_out/c4_12.err; echo "rc=$?" >> gpurun_out/c4_12.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke12.log 2>&1; echo "rc=$?" >> gpurun_out/smoke12.log
tail -n 3 gpurun_out/pytest_gpu12.log
