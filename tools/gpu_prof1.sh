mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bwd_dkdv|k_bwd_dq|attn_fwd2" -s 3 -c 3 -o gpurun_out/prof_k $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
