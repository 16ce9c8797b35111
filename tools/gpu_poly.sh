mkdir -p gpurun_out
for k in 0 2 4 8; do
  VLASIM_POLY=$k timeout -s KILL 300 python tools/bench_attn.py --cfg 4 --iters 20 > gpurun_out/poly_$k.log 2>&1
  echo "poly=$k $(tail -1 gpurun_out/poly_$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["fwd_ms"], d["fp8_fwd_ms"], d["fp8_vs_bf16_max_abs"])')"
done
for k in 4 8; do
VLASIM_POLY=$k timeout -s KILL 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_scale_parity.py -q -m gpu -p no:cacheprovider -x --timeout 300 > gpurun_out/poly_t$k.log 2>&1; echo "tests poly=$k: $(tail -1 gpurun_out/poly_t$k.log)"
done
