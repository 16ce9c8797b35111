# r02 measurement pass: plain bench line, launch list + ncu --set full of the config-2 attention kernels,
# of the config-3 (d = 256) kernels and the config-5 packer launch list.  Each ncu command runs only
# after the same command exited 0 plain.
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs --no-graph --pipeline off"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"attn_fwd2|k_bwd_dkdv|k_bwd_dq|k_bwd_pre" -s 4 -c 4 -o gpurun_out/prof_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu cfg2 rc=$?"
CMD3="python tools/bench_attn.py --cfg 3 --iters 2"
$CMD3 > gpurun_out/plain3.log 2>&1 || { echo "plain cfg3 failed"; tail -5 gpurun_out/plain3.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_p_kernel|k_bwd_dkdv|k_bwd_dq" -s 3 -c 4 -o gpurun_out/prof_cfg3 -f $CMD3 > gpurun_out/ncu_cfg3.log 2>&1
echo "ncu cfg3 rc=$?"
bash tools/gpu_prof_pack.sh
