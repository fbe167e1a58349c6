# round 2, call h: balanced v3 split plan - kernel tests, wave sweep vs the host plan
T=${1:-r2h}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_dataplane_gpu.py tests/test_realtime_gpu.py -m gpu -q --timeout 600 --timeout_method thread > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -n 4 gpurun_out/${T}_tests.log
TF_ATTN_BALANCED=0 timeout 600 python tools/attn_bench.py --batches 32,64,96,128 --plans pool --impls 0 --out gpurun_out/${T}_host.json > gpurun_out/${T}_host.log 2>&1
echo host; grep -h 'c2live560\|short736\|ragged' gpurun_out/${T}_host.log
for w in 1 2 3 4 6; do
  TF_ATTN_BWAVES=$w timeout 600 python tools/attn_bench.py --batches 32,64,96,128 --plans pool --impls 0 --out gpurun_out/${T}_bal_w$w.json > gpurun_out/${T}_bal_w$w.log 2>&1
  echo "balanced waves=$w"; grep -h 'c2live560\|short736\|ragged' gpurun_out/${T}_bal_w$w.log
done
