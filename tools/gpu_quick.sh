mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_cli_capi.py -q -m gpu -p no:cacheprovider --timeout 120 --timeout-method=thread > gpurun_out/t2.log 2>&1; tail -n 3 gpurun_out/t2.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -n 1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'fwd ms', d['roofline']['fwd']['ms'], 'bwd ms', d['roofline']['bwd_ms'], 'TF', d['config']['tflops_effective'])"
VLASIM_PROF=1 timeout -s KILL 300 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep "vlasim prof" | tail -2
