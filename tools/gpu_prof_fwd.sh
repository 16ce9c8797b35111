mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"attn_fwd2_kernel" -s 2 -c 1 -o gpurun_out/prof_fwd3 $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
