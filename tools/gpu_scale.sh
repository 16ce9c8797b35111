# bench.py at N = 1, 2, 4 on one box (torchrun for N > 1), as the driver's scaling run does
mkdir -p gpurun_out
for N in ${NS:-1 2 4}; do
  if [ $N -eq 1 ]; then
    timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/scale_n1.log 2>&1
  else
    timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/scale_n$N.log 2>&1
  fi
  tail -n 1 gpurun_out/scale_n$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'tok/s %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'e2e %.4g' % d['e2e']['value'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
done
