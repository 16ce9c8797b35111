#!/bin/bash
# ncu --set full of the quantizer kernels (one launch each) -> gpurun_out/quant.ncu-rep
cd "$GRAFT_REPO_ROOT" || exit 1
export PYTHONPATH=$PWD:$PYTHONPATH
mkdir -p gpurun_out
timeout -s KILL 300 python tools/quant_prof.py || exit 1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  --kernel-name regex:'k_group_fused|k_tensor_|k_col_' --launch-skip 0 --launch-count 12 \
  -o gpurun_out/quant -f python tools/quant_prof.py > gpurun_out/quant_ncu.log 2>&1
tail -3 gpurun_out/quant_ncu.log
