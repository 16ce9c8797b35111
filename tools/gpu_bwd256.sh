mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_padding.py tests/test_gpu_guard.py tests/test_gpu_seg_src.py -q -m gpu -p no:cacheprovider --timeout 300 -x > gpurun_out/t_attn.log 2>&1; echo "attn: $(tail -n 1 gpurun_out/t_attn.log)"
timeout -s KILL 600 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_shard.py -q -m gpu -p no:cacheprovider --timeout 300 -x > gpurun_out/t_scale.log 2>&1; echo "scale: $(tail -n 1 gpurun_out/t_scale.log)"
timeout -s KILL 300 python tools/bench_attn.py --cfg 3 --iters 10 2>&1 | tail -1
VLASIM_DKV_HALVES=1 timeout -s KILL 300 python tools/bench_attn.py --cfg 3 --iters 10 2>&1 | tail -1
