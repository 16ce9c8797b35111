"""Run config-2-sized bf16 and FP8 forwards and save the outputs (compare two library builds).

  python tools/dbg_cmp_libs.py OUT.pt       (VLASIM_CUDA_LIB selects the library)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11101_b200 import attention, fp8, packing, synthetic

L = synthetic.gen_lengths(512, 0, 16, 512)
plan = packing.pack_ffd(L, 8192)
T, H, d = int(L.sum()), 16, 128
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = (torch.randn(T, H, d, device="cuda", generator=g).bfloat16() for _ in range(3))
seg = packing.seg_src(plan)
o, lse = attention.varlen_attn_fwd(q, k, v, plan.cu_seqlens, seg_src=seg)
qc, qs = fp8.quant_block(q)
kc, ks = fp8.quant_block(k)
o8, _ = fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, plan.cu_seqlens, seg_src=seg)
torch.cuda.synchronize()
torch.save({"o": o.cpu(), "lse": lse.cpu(), "o8": o8.cpu()}, sys.argv[1])
print("saved", (o.float() - o8.float()).abs().max().item())
