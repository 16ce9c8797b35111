# config-3 (d 256) kernels: one ncu --set full capture of the forward and the three backward kernels
mkdir -p gpurun_out
CMD3="python tools/bench_attn.py --cfg 3 --iters 2 --seg-src"
$CMD3 > gpurun_out/plain3.log 2>&1 || { echo "plain cfg3 failed"; tail -5 gpurun_out/plain3.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_p_kernel|k_bwd_dkdv|k_bwd_dq" -s 4 -c 4 -o gpurun_out/prof_cfg3 -f $CMD3 > gpurun_out/ncu_cfg3.log 2>&1
echo "ncu cfg3 rc=$?"
