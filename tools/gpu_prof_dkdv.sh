mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${1:-k_bwd_dkdv}" -s 1 -c 1 -o gpurun_out/prof_dkdv $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
