"""Diagnostic: config-4 FP8 forward timed on bench.py-style vs bench_attn-style inputs, one process."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_11101_b200 import attention, fp8, packing, synthetic  # noqa: E402

dev = torch.device("cuda")
st = torch.cuda.current_stream()
ballast = []
for a in sys.argv:
    if a.startswith("--ballast="):  # GB of live allocations made before the inputs
        ballast = [torch.empty(1 << 30, dtype=torch.uint8, device=dev) for _ in range(int(a.split("=")[1]))]
n = 512
L = synthetic.gen_lengths(n, synthetic.DIST_UNIFORM, 16, 512)
plan = packing.pack_ffd(L, 8192)
T = int(L.sum())
seg = packing.seg_src(plan)
cu = plan.cu_seqlens
q = synthetic.fill_bf16(torch.empty(T, 16, 128, dtype=torch.bfloat16, device=dev), "q")
k = synthetic.fill_bf16(torch.empty(T, 16, 128, dtype=torch.bfloat16, device=dev), "k")
v = synthetic.fill_bf16(torch.empty(T, 16, 128, dtype=torch.bfloat16, device=dev), "v")
res = {}
qc, kc = torch.empty(q.shape, dtype=torch.uint8, device=dev), torch.empty(k.shape, dtype=torch.uint8, device=dev)
qs = torch.empty(16, (T + 127) // 128, 1, dtype=torch.float32, device=dev)
ks = torch.empty_like(qs)
fp8.quant_block(q, codes=qc, scales=qs, check_finite=False)
fp8.quant_block(k, codes=kc, scales=ks, check_finite=False)
qc2, qs2 = fp8.quant_block(q)
kc2, ks2 = fp8.quant_block(k)
res["same_codes"] = bool(torch.equal(qc, qc2) and torch.equal(kc, kc2))
res["same_scales"] = bool(torch.equal(qs, qs2.view_as(qs)) and torch.equal(ks, ks2.view_as(ks)))
res["scale_shapes"] = [list(qs.shape), list(qs2.shape)]
o8, l8 = torch.empty_like(q), torch.empty(16, T, dtype=torch.float32, device=dev)
for tag, (a, b, c, d) in {"bench": (qc, qs, kc, ks), "fresh": (qc2, qs2, kc2, ks2)}.items():
    res[tag] = bench.event_ms(lambda: fp8.varlen_attn_fwd_fp8qk(a, b, c, d, v, cu, out=o8, lse=l8, seg_src=seg),
                              20, st)
o, lse = torch.empty_like(q), torch.empty(16, T, dtype=torch.float32, device=dev)
fws = attention.BwdWorkspace()
res["bf16"] = bench.event_ms(lambda: attention.varlen_attn_fwd(q, k, v, cu, out=o, lse=lse, seg_src=seg,
                                                               workspace=fws), 20, st)
res["bf16_default_ws"] = bench.event_ms(lambda: attention.varlen_attn_fwd(q, k, v, cu, out=o, lse=lse, seg_src=seg),
                                        20, st)
def quant():
    fp8.quant_block(q, codes=qc, scales=qs, check_finite=False)
    fp8.quant_block(k, codes=kc, scales=ks, check_finite=False)


res["quant"] = bench.event_ms(quant, 10, st)
res["after_quant"] = bench.event_ms(lambda: fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, cu, out=o8, lse=l8,
                                                                      seg_src=seg), 10, st)
res["interleaved"] = bench.event_ms(lambda: (quant(), fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, cu, out=o8, lse=l8,
                                                                                 seg_src=seg)), 10, st)
if "--after" in sys.argv:
    rec = []
    orig = fp8.varlen_attn_fwd_fp8qk

    def spy(*a, **kw):
        if not rec:
            rec.append((a, kw))
        return orig(*a, **kw)

    fp8.varlen_attn_fwd_fp8qk = spy
    mc = bench.measure_configs(dev, iters=10)
    fp8.varlen_attn_fwd_fp8qk = orig
    a_, kw_ = rec[0]
    res["recorded_args_retimed"] = bench.event_ms(lambda: orig(*a_, **kw_), 10, st)
    res["recorded_shapes"] = [list(t.shape) for t in a_ if torch.is_tensor(t)]
    res["recorded_kw"] = {k: (list(v.shape) if torch.is_tensor(v) else v) for k, v in kw_.items()}
    res["measure_configs_fp8"] = mc["config4"]["fp8_fwd_ms"]
    res["after_bench"] = bench.event_ms(lambda: fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, cu, out=o8, lse=l8,
                                                                          seg_src=seg), 20, st)
print(json.dumps(res))
