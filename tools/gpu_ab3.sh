# A/B/C of three builds (lib_ab/base.so, c1.so, c2.so) on config 4 (bf16 and FP8 forward), alternating
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in base c1 c2; do
    VLASIM_CUDA_LIB=lib_ab/$v.so timeout -s KILL 300 python tools/bench_attn.py --cfg 4 --iters 20 --seg-src > gpurun_out/ab_$v.log 2>&1
    grep '^{' gpurun_out/ab_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$v'", round(d["fwd_ms"],4), round(d.get("fp8_fwd_ms",0),4))'
  done
done
