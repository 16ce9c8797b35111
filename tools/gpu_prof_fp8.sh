mkdir -p gpurun_out
CMD="python tools/bench_attn.py --cfg 4 --iters 3"
$CMD > gpurun_out/plain4.log 2>&1 || { echo "plain cfg4 failed"; tail -5 gpurun_out/plain4.log; exit 1; }
tail -1 gpurun_out/plain4.log
ncu --set full --clock-control none --import-source on -k regex:"attn_fwd2|k_quant" -s 2 -c 6 -o gpurun_out/prof_cfg4 -f $CMD > gpurun_out/ncu_cfg4.log 2>&1
echo "ncu cfg4 rc=$?"
