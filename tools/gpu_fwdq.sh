mkdir -p gpurun_out
for i in 1 2; do timeout -s KILL 300 python tools/bench_attn.py --cfg 4 --iters 20 > gpurun_out/fwdq_$i.log 2>&1; grep '^{' gpurun_out/fwdq_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("fwd", d["fwd_ms"], "fp8", d["fp8_fwd_ms"], "quant", d["quant_qk_ms"])'; done
timeout -s KILL 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_seg_src.py -q -m gpu -p no:cacheprovider -x --timeout 300 > gpurun_out/fwdq_t.log 2>&1; echo "tests: $(tail -1 gpurun_out/fwdq_t.log)"
