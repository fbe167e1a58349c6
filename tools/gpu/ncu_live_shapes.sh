mkdir -p gpurun_out
for case in 128:ragged500-3000:pool 128:short736:pool; do
  tag=$(echo $case | cut -d: -f1,2 | tr ':' '_')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn -c 1 \
    -o gpurun_out/attn_v3_${tag} -f python tools/attn_bench.py --only $case --reps 1 --out /tmp/x.json \
    > gpurun_out/ncu_attn_v3_${tag}.log 2>&1
done
echo done
