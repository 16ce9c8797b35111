# One ncu --set full capture of the step's attention kernels (fwd, pre, dK/dV, dQ) + launch list.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-graph"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"attn_fwd2|k_bwd_dkdv|k_bwd_dq|k_bwd_pre" -s 4 -c 4 -o gpurun_out/prof_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
