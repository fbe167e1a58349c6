mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_report.py -m gpu -q -x > gpurun_out/rep27a.log 2>&1; echo "rc=$?" >> gpurun_out/rep27a.log
CUDA_LAUNCH_BLOCKING=1 timeout 900 python -m pytest tests/test_report.py -m gpu -q -x > gpurun_out/rep27b.log 2>&1; echo "rc=$?" >> gpurun_out/rep27b.log
TF_ATTN_IMPL=3 timeout 600 python -m pytest tests/test_dataplane_gpu.py -m gpu -q -x -k "replay_parity and not c2" > gpurun_out/rep27c.log 2>&1; echo "rc=$?" >> gpurun_out/rep27c.log
echo done
