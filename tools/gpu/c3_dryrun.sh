mkdir -p gpurun_out
TF_HOST_BLOCKS=8192 TF_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 100 --warmup 5 --no-cpu-baseline --ttft 0 --verbose --graphs 0 > gpurun_out/c3_dry.json 2> gpurun_out/c3_dry.err
echo "rc=$?" >> gpurun_out/c3_dry.err
tail -n 5 gpurun_out/c3_dry.err
