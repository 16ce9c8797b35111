mkdir -p gpurun_out
python tools/pack_cfg5.py > gpurun_out/pack5.log 2>&1 || { tail -5 gpurun_out/pack5.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pack5_launches.csv python tools/pack_cfg5.py > gpurun_out/ncu_pack5.log 2>&1
echo "rc=$?"
