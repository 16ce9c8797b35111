# dK/dV ablations: per-kernel ncu durations with VLASIM_DBG = 0 / 1 (no softmax math) / 2 (no Q/dO
# loads) / 3.  Non-zero values run the PROF instantiation (the only one that honours VLASIM_DBG).
mkdir -p gpurun_out
for D in ${@:-0 1 2 3}; do
  if [ "$D" = "0" ]; then unset VLASIM_PROF; else export VLASIM_PROF=1; fi
  VLASIM_DBG=$D ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bwd_dkdv|k_bwd_dq|attn_fwd2" -s 6 -c 3 --csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu 2>/dev/null | grep gpu__time_duration | \
    awk -F'","' -v d=$D '{split($5,a,"("); printf "dbg=%s %-45s %8.1f us\n", d, substr(a[1],1,45), $NF/1000}' | tr -d '"'
done
unset VLASIM_PROF
