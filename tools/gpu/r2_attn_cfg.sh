T=${1:-r2cfg}
mkdir -p gpurun_out
for c in 0 1; do TF_ATTN5_CFG=$c timeout 300 python tools/attn_bench.py --impls 5 --plans pool --batches 32,64,128 --out gpurun_out/${T}_$c.json 2>&1 | grep -v "uniform\|ragged" | sed "s/^/cfg$c /"; done
TF_ATTN5_CFG=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k attention 2>&1 | tail -2
