"""Fixed-length vs variable-length attention sweep — the paper's varlen experiment (PAPER.md:350-353:
padding rate 3 % → 90 %, seq_len 2k → 32k, batch 8-32) on this repo's sm_100a kernels.

  python tools/bench_padding_sweep.py [--seqs 2048,8192,32768] [--batches 8,16,32]
                                      [--pads 0.03,0.1,0.25,0.5,0.75,0.9] [--heads 16] [--d 128] [--fa2]

For each (seq_len S, batch B, padding rate p): B sample lengths with mean S·(1−p) (uniform around it,
clipped to [1, S]; numpy seed 0).
  fixlen  every sample padded to S: attention fwd+bwd over B segments of S tokens (padded pairs
          computed, like a fixed-length flash-attention call on padded tensors)
  varlen  attention fwd+bwd over the B valid lengths only (cu_seqlens; what packing feeds)
Both run the same hand-written kernels (bidirectional, bf16, H heads × d).  Reported: latencies, the
time saving 1 − varlen/fixlen, TFLOP/s on the pairs each computes (fixlen counts padded pairs,
varlen only valid ones — the paper's convention), and with --fa2 the flash_attn 2.8.3
flash_attn_func / flash_attn_varlen_func times on the same tensors as a comparator.
CUDA-event timing on the launching stream, median of --iters after warm-up.
"""
import argparse
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11101_b200 import attention


def timed(fn, iters):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def lengths(S, B, p, rng):
    m = S * (1.0 - p)
    half = min(m - 1, S - m)  # uniform in [m - half, m + half] ⊂ [1, S]
    L = np.rint(rng.uniform(m - half, m + half, B)).astype(np.int64)
    return np.clip(L, 1, S)


def run_ours(T, H, d, cu, iters, bufs):
    q, k, v, do, o, dq, dk, dv = (x[:T] for x in bufs)
    lse = torch.empty(H, T, dtype=torch.float32, device="cuda")
    ws = attention.BwdWorkspace()

    def fwd():
        attention.varlen_attn_fwd(q, k, v, cu, out=o, lse=lse)

    def fwdbwd():
        attention.varlen_attn_fwd(q, k, v, cu, out=o, lse=lse)
        attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, dq=dq, dk=dk, dv=dv, workspace=ws)
    return timed(fwd, iters), timed(fwdbwd, iters)


def run_fa2(T, H, d, cu, S, B, iters, bufs, fixlen):
    from flash_attn import flash_attn_func, flash_attn_varlen_func
    q, k, v, do = (x[:T].detach().requires_grad_(False) for x in bufs[:4])
    if fixlen:
        qf, kf, vf = (x.view(B, S, H, d).requires_grad_(True) for x in (q.clone(), k.clone(), v.clone()))
        dof = do.view(B, S, H, d)

        def f():
            out = flash_attn_func(qf, kf, vf)
            torch.autograd.backward(out, dof)
    else:
        qv, kv, vv = (x.clone().requires_grad_(True) for x in (q, k, v))
        mx = int((cu[1:] - cu[:-1]).max().item())

        def f():
            out = flash_attn_varlen_func(qv, kv, vv, cu, cu, mx, mx)
            torch.autograd.backward(out, do)
    return timed(f, iters)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", default="2048,8192,32768")
    ap.add_argument("--batches", default="16")
    ap.add_argument("--pads", default="0.03,0.1,0.25,0.5,0.75,0.9")
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--fa2", action="store_true")
    a = ap.parse_args()
    H, d = a.heads, a.d
    seqs = [int(x) for x in a.seqs.split(",")]
    batches = [int(x) for x in a.batches.split(",")]
    pads = [float(x) for x in a.pads.split(",")]
    Tmax = max(seqs) * max(batches)
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda: (torch.randn(Tmax, H, d, device="cuda", generator=g) * 0.5).bfloat16()
    bufs = [mk(), mk(), mk(), mk()] + [torch.empty(Tmax, H, d, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
    rng = np.random.default_rng(0)
    for S in seqs:
        for B in batches:
            iters = a.iters if S * B <= 2 ** 18 else max(2, a.iters // 2)
            cu_fix = torch.arange(0, (B + 1) * S, S, dtype=torch.int32, device="cuda")
            tf_fwd, tf = run_ours(B * S, H, d, cu_fix, iters, bufs)
            fa_fix = run_fa2(B * S, H, d, cu_fix, S, B, iters, bufs, True) if a.fa2 else None
            pairs_fix = float(B) * S * S
            for p in pads:
                L = lengths(S, B, p, rng)
                cu = torch.tensor(np.concatenate([[0], np.cumsum(L)]), dtype=torch.int32, device="cuda")
                T = int(L.sum())
                tv_fwd, tv = run_ours(T, H, d, cu, iters, bufs)
                fa_var = run_fa2(T, H, d, cu, S, B, iters, bufs, False) if a.fa2 else None
                pairs = float(np.sum(L.astype(np.float64) ** 2))
                fl = lambda pr: 3.5 * 4.0 * d * H * pr
                row = {"seq_len": S, "batch": B, "padding_rate": round(1.0 - T / (B * S), 4), "tokens_valid": T,
                       "fixlen_ms": tf, "varlen_ms": tv, "saving": 1.0 - tv / tf,
                       "fixlen_fwd_ms": tf_fwd, "varlen_fwd_ms": tv_fwd,
                       "fixlen_tflops": fl(pairs_fix) / (tf / 1e3) / 1e12,
                       "varlen_tflops": fl(pairs) / (tv / 1e3) / 1e12, "H": H, "d": d, "pass": "fwd+bwd"}
                if a.fa2:
                    row.update({"fa2_fixlen_ms": fa_fix, "fa2_varlen_ms": fa_var, "fa2_saving": 1.0 - fa_var / fa_fix})
                print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
