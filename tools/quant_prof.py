"""Run the general quantizer once per granularity on 8192 x 8192 fp32 (for ncu captures)."""
import torch

from paper_2603_11101_b200 import quant

x = torch.randn(8192, 8192, device="cuda") * torch.logspace(-3, 3, 8192, device="cuda")
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for g, ax in (("tensor", 0), ("channel", 0), ("channel", 1), ("block", 0)):
    for _ in range(2):
        quant.quantize(x, g, ax, check_finite=False, workspace=ws)
torch.cuda.synchronize()
