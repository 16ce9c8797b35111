# Profiling pass (one GPU): plain run, then the launch list, then full captures of the two
# attention kernels.  Each ncu command runs only after the same command exited 0 without ncu.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 3 -c 1 -o gpurun_out/prof_bwd $CMD > gpurun_out/ncu_bwd.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 3 -c 1 -o gpurun_out/prof_fwd $CMD > gpurun_out/ncu_fwd.log 2>&1
echo "rc=$?"
tail -2 gpurun_out/plain.log
