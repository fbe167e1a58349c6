# round 2, call b: new GPU tests (peer all-reduce, host-tier bytes, logits), attention LPT order,
# per-layer vs whole-block swap sweep on the current copy-engine path, C3 dry run WITH graphs
T=${1:-r2b}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
timeout 700 python -m pytest tests/test_dataplane_gpu.py -m gpu -v -x --timeout 600 --durations 0 -k full_size > gpurun_out/${T}_full.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_full.log
tail -n 40 gpurun_out/${T}_full.log
timeout 900 python -m pytest tests/test_ar_gpu.py tests/test_tp_gpu.py tests/test_realtime_gpu.py -m gpu -v --timeout 300 --durations 0 > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -n 15 gpurun_out/${T}_tests.log
timeout 600 python tools/attn_bench.py --batches 64,128 --plans pool --impls 3,5 --orders asis,desc --out gpurun_out/${T}_lpt.json > gpurun_out/${T}_lpt.log 2>&1
TF_ATTN_STAGES=2 timeout 600 python tools/attn_bench.py --batches 64,128 --plans pool --impls 3 --orders asis,desc --out gpurun_out/${T}_lpt_s2.json > gpurun_out/${T}_lpt_s2.log 2>&1
grep -h 'c2live560\|short736' gpurun_out/${T}_lpt.log gpurun_out/${T}_lpt_s2.log
timeout 900 python bench_swap.py --max-blocks 4096 --host-blocks 4096 --engines 1,3 --overlap --out gpurun_out/${T}_swap.json > gpurun_out/${T}_swap.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_swap.log
tail -n 3 gpurun_out/${T}_swap.log
TF_HOST_BLOCKS=8192 TF_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 5 --no-cpu-baseline --ttft 0 --no-selector > gpurun_out/${T}_c3g.json 2> gpurun_out/${T}_c3g.err
echo "rc=$?" >> gpurun_out/${T}_c3g.err
tail -n 5 gpurun_out/${T}_c3g.err; head -c 600 gpurun_out/${T}_c3g.json
