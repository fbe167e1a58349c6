# ncu --set full of v5 at the C2 live shape (tag = $1)
T=${1:-r2ncu}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:paged_attn --launch-skip 5 --launch-count 1 \
    -o gpurun_out/${T}_v5 -f python tools/attn_bench.py --only 128:c2live560:pool --impls 5 --reps 3 --out gpurun_out/${T}_tmp.json > gpurun_out/${T}_ncu.log 2>&1
tail -2 gpurun_out/${T}_ncu.log
