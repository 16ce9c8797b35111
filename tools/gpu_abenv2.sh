# A/B of one build under two environments (base: $ENVV=1, cand: unset), alternating.
# usage: gpu_abenv2.sh CFG [ENVV]   (ENVV defaults to VLASIM_DKV_MODE0)
mkdir -p gpurun_out
CFG=${1:-2}
ENVV=${2:-VLASIM_DKV_MODE0}
for r in 1 2 3 4 5; do
  for v in base cand; do
    if [ $v = base ]; then export $ENVV=1; else unset $ENVV; fi
    timeout -s KILL 300 python tools/bench_attn.py --cfg $CFG --iters 20 --seg-src > gpurun_out/abe_$v.log 2>&1
    grep '^{' gpurun_out/abe_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$v'", round(d["fwd_ms"],4), round(d.get("bwd_ms",0),4))'
  done
done
