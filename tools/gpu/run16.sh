mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu16.log
timeout 700 python bench.py > gpurun_out/bench16.json 2> gpurun_out/bench16.err; echo "rc=$?" >> gpurun_out/bench16.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke16.log 2>&1; echo "rc=$?" >> gpurun_out/smoke16.log
tail -n 3 gpurun_out/pytest_gpu16.log
