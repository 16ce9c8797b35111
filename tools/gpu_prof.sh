# Tests + bench + profiling pass (one GPU).  Each ncu command runs only after the same command
# exited 0 without ncu.
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_attn.py -q -m gpu -p no:cacheprovider --timeout 120 --timeout-method=thread > gpurun_out/t2.log 2>&1; tail -n 3 gpurun_out/t2.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -n 1 gpurun_out/bench.log
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_kernel|attn_fwd2_kernel" -s 6 -c 2 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
