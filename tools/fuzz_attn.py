"""Randomised attention parity sweep against the fp64 oracle (diagnostic; the fixed cases live in
tests/test_gpu_attn.py): random segment counts / lengths (1..700), heads with GQA / MQA groups,
head_dim 64 / 128 / 256, the three masks, both layouts (packed and seg_src).  Prints one line per
case and a summary; exit status 1 on any case outside the north_star tolerance."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as orc_mod  # noqa: E402
from paper_2603_11101_b200 import attention  # noqa: E402

TOL = 2e-2


def err(x, ref):
    x = x.float().cpu().numpy().astype(np.float64)
    return float(np.max(np.abs(x - ref)) / max(1.0, np.max(np.abs(ref))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=40)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    orc = orc_mod
    rng = np.random.default_rng(a.seed)
    worst, bad = 0.0, 0
    for c in range(a.cases):
        d = int(rng.choice([64, 128, 256]))
        hkv = int(rng.choice([1, 2]))
        H = hkv * int(rng.choice([1, 2, 4] if d < 256 else [1, 4, 8]))
        mask = int(rng.integers(0, 3))
        n = int(rng.integers(1, 9))
        L = [int(x) for x in rng.integers(1, 700, n)]
        T = sum(L)
        g = torch.Generator(device="cuda").manual_seed(c)
        q = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
        k = torch.randn(T, hkv, d, device="cuda", generator=g).bfloat16()
        v = torch.randn(T, hkv, d, device="cuda", generator=g).bfloat16()
        do = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
        cu = torch.tensor(np.concatenate([[0], np.cumsum(L)]), dtype=torch.int32, device="cuda")
        prefix = torch.tensor([int(rng.integers(0, l + 1)) for l in L], dtype=torch.int32, device="cuda") \
            if mask == 2 else None
        o, lse = attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix)
        dq, dk, dv = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, mask_mode=mask, prefix_len=prefix)
        torch.cuda.synchronize()
        f = lambda t: t.float().cpu().numpy()  # noqa: E731
        pre = None if prefix is None else prefix.cpu().numpy()
        ro, _ = orc.mha_fwd(f(q), f(k), f(v), cu.cpu().numpy(), mask=mask, prefix=pre)
        rdq, rdk, rdv = orc.mha_bwd(f(q), f(k), f(v), ro, f(do), cu.cpu().numpy(), mask=mask, prefix=pre)
        e = max(err(o, ro), err(dq, rdq), err(dk, rdk), err(dv, rdv))
        worst = max(worst, e)
        ok = e < TOL
        bad += not ok
        print(f"case {c:3d} n={n} T={T:5d} H={H} Hkv={hkv} d={d} mask={mask} max_err={e:.2e} {'ok' if ok else 'FAIL'}",
              flush=True)
    print(f"summary: {a.cases} cases, worst {worst:.2e}, failures {bad}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
