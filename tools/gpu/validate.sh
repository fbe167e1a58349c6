mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu31.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu31.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke31.log 2>&1; echo "rc=$?" >> gpurun_out/smoke31.log
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench31.json 2> gpurun_out/bench31.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/bench31.err
tail -n 3 gpurun_out/pytest_gpu31.log
