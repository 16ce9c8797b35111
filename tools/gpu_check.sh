# Full GPU check: every -m gpu test file separately (bounded), smoke, the default bench line.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
for f in tests/test_gpu_*.py tests/test_cli_capi.py tests/test_cli_config.py tests/test_dropin_cpp.py tests/test_bench_contract.py; do
  b=$(basename $f .py)
  timeout -s KILL 900 python -m pytest $f -q -m gpu -p no:cacheprovider --timeout 600 --timeout-method=thread > gpurun_out/$b.log 2>&1
  echo "$b: $(tail -n 1 gpurun_out/$b.log)"
done
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -n 1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 4000 gpurun_out/bench.log
