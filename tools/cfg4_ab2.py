"""Diagnostic: bf16 / FP8 forward on fresh buffers allocated before and after bench.measure_configs."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_11101_b200 import attention, fp8, packing, synthetic  # noqa: E402

dev = torch.device("cuda")
st = torch.cuda.current_stream()


def case():
    L = synthetic.gen_lengths(512, synthetic.DIST_UNIFORM, 16, 512)
    plan = packing.pack_ffd(L, 8192)
    T = int(L.sum())
    seg = packing.seg_src(plan)
    cu = plan.cu_seqlens
    q = synthetic.fill_bf16(torch.empty(T, 16, 128, dtype=torch.bfloat16, device=dev), "q")
    k = synthetic.fill_bf16(torch.empty(T, 16, 128, dtype=torch.bfloat16, device=dev), "k")
    v = synthetic.fill_bf16(torch.empty(T, 16, 128, dtype=torch.bfloat16, device=dev), "v")
    qc, qs = fp8.quant_block(q)
    kc, ks = fp8.quant_block(k)
    o, lse = torch.empty_like(q), torch.empty(16, T, dtype=torch.float32, device=dev)
    fws = attention.BwdWorkspace()
    f16 = lambda: attention.varlen_attn_fwd(q, k, v, cu, out=o, lse=lse, seg_src=seg, workspace=fws)  # noqa: E731
    f8 = lambda: fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, cu, out=o, lse=lse, seg_src=seg)  # noqa: E731
    return f16, f8


res = {}
a16, a8 = case()
res["before"] = bench.ab_ms(a8, a16, 20, st)
mc = bench.measure_configs(dev, iters=10)
res["measure_configs"] = (mc["config4"]["fp8_fwd_ms"], mc["config4"]["bf16_fwd_ms"])
res["old_buffers_after"] = bench.ab_ms(a8, a16, 20, st)
b16, b8 = case()
res["new_buffers_after"] = bench.ab_ms(b8, b16, 20, st)
print(json.dumps(res))
