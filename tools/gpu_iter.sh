# Iteration pass: attention / fp8 / C-ABI GPU tests, attention-only timing (configs 2-4), bench step.
mkdir -p gpurun_out
timeout -s KILL 500 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_cli_capi.py -q -m gpu -x -p no:cacheprovider --timeout 120 --timeout-method=thread > gpurun_out/t2.log 2>&1; tail -n 15 gpurun_out/t2.log
for c in 2 3 4; do timeout -s KILL 200 python tools/bench_attn.py --cfg $c > gpurun_out/attn_cfg$c.log 2>&1; tail -n 3 gpurun_out/attn_cfg$c.log; done
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -n 1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'fwd ms', d['roofline']['fwd']['ms'], 'bwd ms', d['roofline']['bwd_ms'], 'TF', d['config']['tflops_effective'])"
