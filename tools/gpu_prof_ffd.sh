mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
ncu -f --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"k_ffd_warp" -s 3 -c 1 -o gpurun_out/prof_ffd $CMD > gpurun_out/ncu_ffd.log 2>&1
echo "rc=$?"
