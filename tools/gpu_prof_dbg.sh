# ncu full capture of the dK/dV kernel under VLASIM_DBG=$1 (timing ablations)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
VLASIM_DBG=$1 $CMD > gpurun_out/plain.log 2>&1 && \
VLASIM_DBG=$1 ncu --set full --clock-control none --import-source on -k regex:k_bwd_dkdv -s 1 -c 1 -o gpurun_out/prof_dbg$1 $CMD > gpurun_out/ncu_dbg.log 2>&1
echo "rc=$?"
