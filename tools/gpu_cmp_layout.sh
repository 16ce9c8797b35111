# bench step variants (fused / packed layout, pipelined pack on / off), one line each
for v in "--pipeline on" "--pipeline off" "--layout packed"; do
  timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e $v > gpurun_out/bench_var.log 2>&1
  tail -n 1 gpurun_out/bench_var.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', 'ms/step', round(d['ms_per_step'],4), 'pack', round(r['pack_ms'],4), 'fwd', round(r['fwd']['ms'],4), 'bwd', round(r['bwd_ms'],4), 'Mtok/s', round(d['value']/1e6,2))" || tail -5 gpurun_out/bench_var.log
done
