#!/bin/bash
# FP8 forward with and without seg_src (sample-major inputs), then one ncu capture of each
cd "$GRAFT_REPO_ROOT" || exit 1
export PYTHONPATH=$PWD:$PYTHONPATH
mkdir -p gpurun_out
for m in "" "--seg-src"; do
  timeout -s KILL 300 python tools/bench_attn.py --cfg 4 --iters 20 $m > gpurun_out/fp8seg.log 2>&1
  grep '^{' gpurun_out/fp8seg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("seg_src", d["seg_src"], "fwd", d["fwd_ms"], "fp8", d["fp8_fwd_ms"])'
done
for m in "" "--seg-src"; do
  tag=$([ -z "$m" ] && echo packed || echo seg)
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd2 -s 8 -c 1 \
    -o gpurun_out/fp8_$tag -f python tools/bench_attn.py --cfg 4 --iters 2 $m > gpurun_out/ncu_fp8_$tag.log 2>&1
  echo "ncu $tag rc=$?"
done
