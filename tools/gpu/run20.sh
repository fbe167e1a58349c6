mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu20.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu20.log
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench20.json 2> gpurun_out/bench20.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/bench20.err
timeout 700 python bench.py --profile-hooks --no-cpu-baseline > gpurun_out/bench20h.json 2> gpurun_out/bench20h.err
tail -n 3 gpurun_out/pytest_gpu20.log
