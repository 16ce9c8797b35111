mkdir -p gpurun_out
CMD="python tools/bench_attn.py --cfg 4 --iters 2"
$CMD > gpurun_out/plain4.log 2>&1 || { echo "plain cfg4 failed"; tail -5 gpurun_out/plain4.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:attn_fwd2 -s 6 -c 1 -o gpurun_out/prof_fp8 -f $CMD > gpurun_out/ncu_fp8.log 2>&1
echo "ncu fp8 rc=$?"
