# GPU tests (attention) + bench + ncu launch list + ncu full capture of the attention kernels
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_attn.py -q -m gpu -p no:cacheprovider --timeout 120 --timeout-method=thread > gpurun_out/t2.log 2>&1; tail -n 2 gpurun_out/t2.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -n 1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'fwd ms', d['roofline']['fwd']['ms'], 'bwd ms', d['roofline']['bwd_ms'], 'TF', d['config']['tflops_effective'])"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"attn_fwd2|k_bwd_pre|k_bwd_dkdv|k_bwd_dq" -s 8 -c 4 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
