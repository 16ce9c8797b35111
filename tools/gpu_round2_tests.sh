# GPU test pass: every -m gpu test file separately (bounded), smoke, one bench line.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
for f in tests/test_gpu_*.py tests/test_cli_capi.py; do
  b=$(basename $f .py)
  timeout -s KILL 600 python -m pytest $f -q -m gpu -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/$b.log 2>&1
  echo "$b: $(tail -n 1 gpurun_out/$b.log)"
done
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -n 1 gpurun_out/smoke.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
tail -n 1 gpurun_out/bench.log
