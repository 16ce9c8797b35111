# 2-GPU checks: the union-of-shards test under torchrun, then bench.py at N = 2 (DDP block included).
mkdir -p gpurun_out
N=${1:-2}
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tools/mgpu_union.py gpurun_out/mgpu_union_$N.json > gpurun_out/mgpu_union_$N.log 2>&1; echo "union rc=$?"; tail -2 gpurun_out/mgpu_union_$N.log
timeout -s KILL 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_n$N.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_n$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d.get('ddp_allreduce')))"
