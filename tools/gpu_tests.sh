mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_umma.py tests/test_gpu_pack.py -q -m gpu -p no:cacheprovider --timeout 120 --timeout-method=thread > gpurun_out/t1.log 2>&1
timeout -s KILL 400 python -m pytest tests/test_gpu_attn.py -q -m gpu -p no:cacheprovider --timeout 120 --timeout-method=thread > gpurun_out/t2.log 2>&1
tail -n 3 gpurun_out/t1.log; tail -n 3 gpurun_out/t2.log
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -n 2 gpurun_out/smoke.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
tail -n 3 gpurun_out/bench.log
