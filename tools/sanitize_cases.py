"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): packer (FFD + greedy + token ids + gather/scatter), attention fwd/bwd for head_dim 64 /
128 / 256 and the three masks (packed and seg_src layouts), FP8 quantiser + FP8 forward/backward,
the general quantizer, dynamic padding and the shard plan.  Exit 0 when every call returned."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_11101_b200 import attention, dist as vdist, fp8, packing, padding, quant, synthetic  # noqa: E402


def main():
    dev = torch.device("cuda")
    L = synthetic.gen_lengths(24, synthetic.DIST_UNIFORM, 1, 300, seed=3)
    plan = packing.pack_ffd(L, 1024)
    packing.pack_greedy(L, 1024)
    T = int(L.sum())
    pos, seg, gat = packing.token_ids(plan, T)
    x = torch.randn(T, 2, 64, device=dev).bfloat16()
    packing.scatter_rows(packing.gather_rows(x, plan), plan)
    vdist.shard_lpt(plan, 2, 1)
    cu = plan.cu_seqlens
    segsrc = packing.seg_src(plan)
    for H, Hkv, d in ((2, 2, 64), (4, 2, 128), (4, 1, 256)):
        for mask in (0, 1, 2):
            q, do = (torch.randn(T, H, d, device=dev).bfloat16() for _ in range(2))
            k, v = (torch.randn(T, Hkv, d, device=dev).bfloat16() for _ in range(2))
            pre = torch.full((L.size,), 40, dtype=torch.int32, device=dev) if mask == 2 else None
            for ss in (None, segsrc):
                o, lse = attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=pre, seg_src=ss)
                attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, mask_mode=mask, prefix_len=pre, seg_src=ss)
            torch.cuda.synchronize()
    q, do = (torch.randn(T, 4, 128, device=dev).bfloat16() for _ in range(2))
    k, v = (torch.randn(T, 4, 128, device=dev).bfloat16() for _ in range(2))
    qc, qs = fp8.quant_block(q)
    kc, ks = fp8.quant_block(k)
    o8, l8 = fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, cu)
    fp8.varlen_attn_bwd_fp8qk(do, qc, qs, kc, ks, v, o8, l8, cu)
    fp8.quant_error(q, qc, qs)
    w = torch.randn(300, 260, device=dev)
    for g, ax in (("tensor", 0), ("channel", 1), ("block", 0)):
        qt = quant.quantize(w, g, ax)
        quant.dequantize(qt)
        quant.quant_error(w, qt)
    dp = padding.dynamic_pad(L)
    qp = padding.pad_rows(q, dp)
    padding.unpad_rows(qp, dp)
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
