# A/B of two builds of libvlasim_cuda.so on the same box (lib_ab/base.so vs lib_ab/cand.so), alternating
mkdir -p gpurun_out
CFG=${1:-2}
SEG=${2:-}
for r in 1 2 3; do
  for v in base cand; do
    VLASIM_CUDA_LIB=lib_ab/$v.so timeout -s KILL 300 python tools/bench_attn.py --cfg $CFG --iters 20 $SEG > gpurun_out/ab_$v.log 2>&1
    grep '^{' gpurun_out/ab_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$v'", round(d["fwd_ms"],4), round(d.get("bwd_ms",0),4), round(d.get("fp8_fwd_ms",0),4), round(d.get("quant_qk_ms",0),4))'
  done
done
