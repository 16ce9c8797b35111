"""Config-5 packer run for profiling: 1M samples, truncated geometric(p=0.02, max 500) lengths, cap 8192."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_11101_b200 import dist as vdist, packing, synthetic  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
L = torch.from_numpy(synthetic.gen_lengths(n, synthetic.DIST_GEOMETRIC, 0.02, 500)).cuda()
plan = packing.pack_ffd(L, 8192)
for _ in range(3):
    packing.pack_ffd(L, 8192, plan=plan, sync_check=False)
    vdist.shard_lpt(plan, 8, 0, sync_check=False)
torch.cuda.synchronize()
print("bins", plan.num_bins())
