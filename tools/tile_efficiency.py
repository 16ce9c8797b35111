"""Computed-pair efficiency of the attention tilings on the config-2 packs (CPU only).

  python tools/tile_efficiency.py [--samples 512] [--capacity 8192]

valid pairs = Σ l² (bidirectional); computed pairs = what the kernels multiply for each tiling.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import oracle
from paper_2603_11101_b200.synthetic import gen_lengths


def rup(x, g):
    return -(-x // g) * g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=512)
    ap.add_argument("--capacity", type=int, default=8192)
    a = ap.parse_args()
    L = gen_lengths(a.samples, 0, 16, 512, seed=42, label="lengths")
    b, s, t, nb = oracle.pack(L, a.capacity, 1)
    cu = oracle.layout(L, b, s, t, nb)["cu_seqlens"]
    T = int(cu[-1])
    seglen = np.diff(cu)
    segid = np.repeat(np.arange(len(seglen)), seglen)
    lo, hi = cu[segid], cu[segid + 1]
    V = float((seglen.astype(np.float64) ** 2).sum())
    grid = sum(128 * rup(hi[min(q0 + 127, T - 1)] - lo[q0], 128) for q0 in range(0, T, 128))
    print(f"Q tiles on the 128-row grid, 128-key tiles:        {V / grid:.3f}")
    for g in (128, 32):
        c = sum(-(-l // 128) * 128 * ((l // 128) * 128 + (rup(l % 128, g) if l % 128 else 0)) for l in seglen)
        print(f"segment-aligned Q tiles, last key tile N%{g:<3d}:      {V / c:.3f}")
    kv = sum(128 * rup(hi[min(k0 + 127, T - 1)] - lo[k0], 64) for k0 in range(0, T, 128))
    print(f"dK/dV, key tiles on the grid, 64-query units:      {V / kv:.3f}")
    kv = sum(-(-l // 128) * 128 * rup(l, 64) for l in seglen)
    print(f"dK/dV, segment-aligned key tiles, 64-query units:  {V / kv:.3f}")


if __name__ == "__main__":
    main()
