T=${1:-r2swap}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k swap > gpurun_out/${T}_tests.log 2>&1; tail -2 gpurun_out/${T}_tests.log
timeout 300 python bench_swap.py --wt-only --out gpurun_out/${T}_wt.json 2>&1 | tail -60
