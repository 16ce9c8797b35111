# Full measurement pass: GPU tests, smoke, default bench (e2e + CPU baseline), reference arm,
# layout / pipeline variants, ncu launch list and one --set full capture of the attention kernels.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; python -c "import os; print(len(os.sched_getaffinity(0)))" >> gpurun_out/nproc.txt
timeout -s KILL 600 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/tests_gpu.log 2>&1; tail -n 2 gpurun_out/tests_gpu.log
timeout -s KILL 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -n 1 gpurun_out/smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -n 1 gpurun_out/bench_default.log
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -n 1 gpurun_out/bench_ref.log
timeout -s KILL 300 python bench.py --dist groot --no-cpu --no-e2e > gpurun_out/bench_groot.log 2>&1; tail -n 1 gpurun_out/bench_groot.log
timeout -s KILL 300 python bench.py --pipeline off --no-cpu --no-e2e > gpurun_out/bench_nopipe.log 2>&1; tail -n 1 gpurun_out/bench_nopipe.log
timeout -s KILL 300 python bench.py --layout packed --no-cpu --no-e2e > gpurun_out/bench_packed.log 2>&1; tail -n 1 gpurun_out/bench_packed.log
for c in 2 3 4; do timeout -s KILL 200 python tools/bench_attn.py --cfg $c > gpurun_out/attn_cfg$c.log 2>&1; tail -n 1 gpurun_out/attn_cfg$c.log; done
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"attn_fwd2|k_bwd_dkdv|k_bwd_dq|k_bwd_pre|k_ffd_warp" -s 5 -c 5 -o gpurun_out/prof_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
