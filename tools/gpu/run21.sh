mkdir -p gpurun_out
for i in 1 2; do t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench21_$i.json 2> gpurun_out/bench21_$i.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/bench21_$i.err; done
echo done
