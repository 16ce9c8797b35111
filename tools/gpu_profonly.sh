mkdir -p gpurun_out
VLASIM_PROF=1 timeout -s KILL 300 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep "vlasim prof" | tail -2
