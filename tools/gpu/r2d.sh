# diagnose the C2 full-size replay stall: default attention with a thread-method timeout (stack dump),
# then the same test with v3 attention forced
T=${1:-r2d}
mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_dataplane_gpu.py -m gpu -v -x --timeout 360 --timeout_method thread -k full_size > gpurun_out/${T}_v5.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_v5.log
tail -n 60 gpurun_out/${T}_v5.log
TF_ATTN_IMPL=3 timeout 900 python -m pytest tests/test_dataplane_gpu.py -m gpu -v -x --timeout 800 --timeout_method thread --durations 3 -k full_size > gpurun_out/${T}_v3.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_v3.log
tail -n 30 gpurun_out/${T}_v3.log
