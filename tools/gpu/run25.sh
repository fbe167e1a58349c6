mkdir -p gpurun_out
TF_ATTN_WARPS=2 timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -k attention > gpurun_out/pytest_w2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_w2.log
for w in 2 4; do TF_ATTN_WARPS=$w timeout 300 python tools/attn_bench.py --out gpurun_out/attn_w$w.json > /dev/null 2>&1; done
echo done
