mkdir -p gpurun_out
for f in tests/test_gpu_shard.py tests/test_dropin_cpp.py tests/test_gpu_attn.py tests/test_bench_contract.py; do
  b=$(basename $f .py)
  timeout -s KILL 600 python -m pytest $f -q -m gpu -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/$b.log 2>&1
  echo "$b: $(tail -n 1 gpurun_out/$b.log)"
done
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -c 6000 gpurun_out/bench_default.log
