"""Bisect helper: run one small backward with VLASIM_BWD_DEBUG=<mask> and report the outcome."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2603_11101_b200 import attention
L = [100, 28, 300, 5, 1, 130]
T, H, d = sum(L), 2, 128
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn(T, H, d, device="cuda", generator=g).bfloat16() for _ in range(4))
cu = torch.tensor(np.concatenate([[0], np.cumsum(L)]), dtype=torch.int32, device="cuda")
o, lse = attention.varlen_attn_fwd(q, k, v, cu)
torch.cuda.synchronize()
print("fwd ok", flush=True)
try:
    dq, dk, dv = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu)
    torch.cuda.synchronize()
    print("mask", os.environ.get("VLASIM_BWD_DEBUG"), "OK", float(dq.float().abs().max()), float(dk.float().abs().max()))
except Exception as e:
    print("mask", os.environ.get("VLASIM_BWD_DEBUG"), "FAIL", str(e).splitlines()[0])
