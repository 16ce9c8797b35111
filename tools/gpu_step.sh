# attention tests + kernel times (config 2, config 3) + one default-ish bench line
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_padding.py tests/test_gpu_guard.py tests/test_gpu_seg_src.py tests/test_gpu_fp8.py tests/test_gpu_scale_parity.py tests/test_gpu_shard.py -q -m gpu -p no:cacheprovider --timeout 300 -x > gpurun_out/t_step.log 2>&1; echo "tests: $(tail -n 1 gpurun_out/t_step.log)"
for c in 2 3; do timeout -s KILL 300 python tools/bench_attn.py --cfg $c --iters 20 > gpurun_out/step_cfg$c.log 2>&1; grep '^{' gpurun_out/step_cfg$c.log; done
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-configs > gpurun_out/step_bench.log 2>&1; tail -1 gpurun_out/step_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("bench", d["value"], d["ms_per_step"], d["kernel_ms"])'
