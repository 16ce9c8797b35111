mkdir -p gpurun_out
for v in new halves; do
  if [ $v = halves ]; then export VLASIM_DKV_HALVES=1; fi
  ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum.per_second --clock-control none -k regex:k_bwd --csv python tools/bench_attn.py --cfg 3 --iters 1 2>/dev/null | grep -E "k_bwd" | awk -F'","' '{print $5" | "$13" | "$15}' | sed 's/(CUtensorMap_st.*BwdParams)//' | tail -12 > gpurun_out/bwd256_$v.txt
  echo "== $v"; cat gpurun_out/bwd256_$v.txt | tail -12
done
