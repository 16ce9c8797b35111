"""Quantizer timing per granularity (8192 x 8192 fp32 and bf16, preallocated outputs, CUDA events,
median of 20) for same-box A/B of two builds (VLASIM_CUDA_LIB)."""
import json
import statistics

import torch

from paper_2603_11101_b200 import quant

res = {}
for dt in (torch.float32, torch.bfloat16):
    x = (torch.randn(8192, 8192, device="cuda") * torch.logspace(-3, 3, 8192, device="cuda")).to(dt)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for g, ax in (("tensor", 0), ("channel", 0), ("channel", 1), ("block", 0)):
        out = quant.quantize(x, g, ax, check_finite=False, workspace=ws)
        ts = []
        for i in range(23):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            quant.quantize(x, g, ax, check_finite=False, workspace=ws, out=out)
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        res[f"{str(dt)[6:]}:{g}:{ax}"] = round(statistics.median(ts), 1)
print(json.dumps(res))
