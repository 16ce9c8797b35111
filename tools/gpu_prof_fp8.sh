# FP8 vs bf16 forward at config-2 scale: PROF wait counters and one ncu --set full capture of each
mkdir -p gpurun_out
CMD="python tools/bench_attn.py --cfg 4 --iters 2 --seg-src"
$CMD > gpurun_out/plain4.log 2>&1 || { echo "plain cfg4 failed"; tail -5 gpurun_out/plain4.log; exit 1; }
VLASIM_PROF=1 timeout -s KILL 200 $CMD 2>&1 | grep -E "attn_fwd2" | sort | uniq -c
ncu --set full --clock-control none --import-source on -k regex:attn_fwd2 -s 2 -c 1 -o gpurun_out/prof_bf16f -f $CMD > gpurun_out/ncu_bf16f.log 2>&1
echo "ncu bf16 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:attn_fwd2 -s 6 -c 1 -o gpurun_out/prof_fp8 -f $CMD > gpurun_out/ncu_fp8.log 2>&1
echo "ncu fp8 rc=$?"
