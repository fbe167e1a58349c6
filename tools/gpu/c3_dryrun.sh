mkdir -p gpurun_out
TF_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 200 --warmup 5 --no-cpu-baseline --ttft 1 > gpurun_out/c3_dry.json 2> gpurun_out/c3_dry.err
echo "rc=$?" >> gpurun_out/c3_dry.err
TF_BENCH_ONE_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 --cpu-seconds 3 > gpurun_out/c3_ref.json 2> gpurun_out/c3_ref.err
echo "rc=$?" >> gpurun_out/c3_ref.err
tail -n 3 gpurun_out/c3_dry.err
