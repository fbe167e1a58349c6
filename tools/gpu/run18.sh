mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tp_gpu.py -m gpu -q > gpurun_out/pytest_tp18.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tp18.log
timeout 700 python bench.py > gpurun_out/bench18.json 2> gpurun_out/bench18.err; echo "rc=$?" >> gpurun_out/bench18.err
timeout 900 python bench.py --config c4 --steps 200 --no-cpu-baseline > gpurun_out/c4_18.json 2> gpurun_out/c4_18.err; echo "rc=$?" >> gpurun_out/c4_18.err
tail -n 3 gpurun_out/pytest_tp18.log
