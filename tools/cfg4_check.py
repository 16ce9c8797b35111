"""Config-4 FP8 forward timed as bench.py's measure_configs does, standalone (diagnostic)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

dev = torch.device("cuda")

out = bench.measure_configs(dev, iters=10)
print(json.dumps({"config4": {k: out["config4"][k] for k in ("fp8_fwd_ms", "bf16_fwd_ms", "quant_qk_ms")},
                  "config2_fwd": out["config2_kernels"]["kernel_ms"] if "config2_kernels" in out else None}))
