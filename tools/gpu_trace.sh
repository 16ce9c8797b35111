# CTA-0 event trace of the dK/dV kernel (PROF build; VLASIM_DBG must include 2 — see attn_bwd.cu)
mkdir -p gpurun_out
rm -f gpurun_out/trace.bin
VLASIM_DBG=${1:-2} VLASIM_PROF=1 VLASIM_TRACE=gpurun_out/trace.bin timeout -s KILL 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e 2>&1 | grep "vlasim prof" | tail -1
