mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -k launch_counter > gpurun_out/pytest32.log 2>&1; echo "rc=$?" >> gpurun_out/pytest32.log
timeout 700 python bench.py --arrivals poisson --full-run --no-cpu-baseline --max-wall 500 > gpurun_out/full32p.json 2> gpurun_out/full32p.err; echo "rc=$?" >> gpurun_out/full32p.err
echo done
