mkdir -p gpurun_out
for m in 0 1 2 4 8 16 32 14 62 63; do
  VLASIM_BWD_DEBUG=$m timeout -s KILL 60 python tools/dbg_bwd.py 2>&1 | grep -E "mask|Error|error" | head -2
done
timeout -s KILL 400 python -m pytest tests/test_gpu_pack.py -q -m gpu -p no:cacheprovider --timeout 120 --timeout-method=thread 2>&1 | tail -3
