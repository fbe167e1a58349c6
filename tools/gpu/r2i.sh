# round 2, call i: v3 L2 bulk prefetch past the ring (TF_ATTN_PF) on the host plan
T=${1:-r2i}
mkdir -p gpurun_out
for pf in 0 1 2 4; do
  TF_ATTN_PF=$pf timeout 600 python tools/attn_bench.py --batches 32,64,96,128 --plans pool --impls 0 --out gpurun_out/${T}_pf$pf.json > gpurun_out/${T}_pf$pf.log 2>&1
  echo "pf=$pf"; grep -h 'c2live560\|short736\|ragged\|uniform' gpurun_out/${T}_pf$pf.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['B'],d['ctx'],d['us'],d['frac'])"
done
TF_ATTN_PF=2 timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -k paged_attention > gpurun_out/${T}_tests.log 2>&1; tail -n 2 gpurun_out/${T}_tests.log
