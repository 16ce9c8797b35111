mkdir -p gpurun_out
for f in tests/test_gpu_pack.py tests/test_gpu_fp8.py; do
  b=$(basename $f .py)
  timeout -s KILL 900 python -m pytest $f -q -m gpu -p no:cacheprovider --timeout 600 -x > gpurun_out/$b.log 2>&1
  echo "$b: $(tail -n 3 gpurun_out/$b.log)"
done
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['configs']['config4'])[:900], json.dumps(d['configs']['config5']))"
