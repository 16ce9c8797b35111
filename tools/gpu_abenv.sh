# A/B of an environment switch on the same library and box
mkdir -p gpurun_out
CFG=${1:-2}; VAR=$2
for r in 1 2 3; do
  for v in off on; do
    if [ $v = on ]; then export $VAR=1; else unset $VAR; fi
    timeout -s KILL 300 python tools/bench_attn.py --cfg $CFG --iters 20 > gpurun_out/abe_$v.log 2>&1
    grep '^{' gpurun_out/abe_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$v'", round(d["fwd_ms"],4), round(d.get("bwd_ms",0),4))'
  done
done
