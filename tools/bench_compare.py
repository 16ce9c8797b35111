"""Library comparators on identical packs ("FA2 2.8.3 varlen GPU time on identical
packs is reported as a comparator").  Not part of the product or of bench.py's contract line.

  python tools/bench_compare.py [--cfg 2|3]

Times, with CUDA events after warm-up (median of --iters):
  ours        vlasim varlen fwd / bwd (this repo's sm_100a kernels)
  fa2         flash_attn 2.8.3 flash_attn_varlen_func fwd / bwd (if it runs on this GPU)
  flashinfer  flashinfer BatchPrefillWithRaggedKVCacheWrapper fwd (if it runs on this GPU)
and the max-abs difference of each comparator's O against ours.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11101_b200 import attention, packing, synthetic


def timed(fn, iters):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2, choices=[2, 3])
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda")
    if a.cfg == 3:
        L = synthetic.gen_lengths(256, synthetic.DIST_PI05, 16, 200, 50)
        H, Hkv, d, mask = 8, 1, 256, 2
    else:
        L = synthetic.gen_lengths(512, synthetic.DIST_UNIFORM, 16, 512)
        H, Hkv, d, mask = 16, 16, 128, 0
    n = len(L)
    plan = packing.pack_ffd(L, 8192)
    T = plan.total_tokens()
    Lp = L[plan.member_ids[:n].cpu().numpy()]
    prefix_h = np.maximum(Lp - 50, 0).astype(np.int32) if mask == 2 else None
    prefix = torch.from_numpy(prefix_h).to(dev) if mask == 2 else None
    pairs = packing.visible_pairs(Lp.tolist(), mask, None if prefix_h is None else prefix_h.tolist())
    fl = 4.0 * d * H * pairs
    q = synthetic.fill_bf16(torch.empty(T, H, d, dtype=torch.bfloat16, device=dev), "q")
    k = synthetic.fill_bf16(torch.empty(T, Hkv, d, dtype=torch.bfloat16, device=dev), "k")
    v = synthetic.fill_bf16(torch.empty(T, Hkv, d, dtype=torch.bfloat16, device=dev), "v")
    do = synthetic.fill_bf16(torch.empty(T, H, d, dtype=torch.bfloat16, device=dev), "do")
    cu = plan.cu_seqlens[: n + 1].contiguous()
    out = {"cfg": a.cfg, "tokens": T, "H": H, "Hkv": Hkv, "d": d, "mask": mask, "fwd_tflop": fl / 1e12}
    o = torch.empty_like(q)
    lse = torch.empty(H, T, dtype=torch.float32, device=dev)
    ws = attention.BwdWorkspace()
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    tf = timed(lambda: attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix, out=o, lse=lse),
               a.iters)
    tb = timed(lambda: attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, mask_mode=mask, prefix_len=prefix,
                                                 workspace=ws, dq=dq, dk=dk, dv=dv), a.iters)
    out["ours"] = {"fwd_ms": tf, "bwd_ms": tb, "fwd_tflops": fl / tf / 1e9, "bwd_tflops": 2.5 * fl / tb / 1e9}
    maxlen = int(Lp.max())
    causal = mask != 0
    if mask == 2:  # the comparators have no prefix mask: all three are also timed causal
        cpairs = packing.visible_pairs(Lp.tolist(), 1)
        fl = 4.0 * d * H * cpairs
        tf = timed(lambda: attention.varlen_attn_fwd(q, k, v, cu, mask_mode=1, out=o, lse=lse), a.iters)
        tb = timed(lambda: attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, mask_mode=1, workspace=ws, dq=dq,
                                                     dk=dk, dv=dv), a.iters)
        out["ours_causal"] = {"fwd_ms": tf, "bwd_ms": tb, "fwd_tflops": fl / tf / 1e9,
                              "bwd_tflops": 2.5 * fl / tb / 1e9}
        out["note"] = "fa2 / flashinfer have no prefix mask: compare them with ours_causal"
    try:
        from flash_attn import flash_attn_varlen_func
        qq, kk, vv = (x.detach().clone().requires_grad_(True) for x in (q, k, v))

        def fa_fwd():
            return flash_attn_varlen_func(qq, kk, vv, cu, cu, maxlen, maxlen, causal=causal)

        with torch.no_grad():
            tf2 = timed(fa_fwd, a.iters)
            of = fa_fwd()
        ofa = fa_fwd()

        def fa_bwd():
            torch.autograd.grad(ofa, (qq, kk, vv), do, retain_graph=True)

        tb2 = timed(fa_bwd, a.iters)
        out["fa2"] = {"fwd_ms": tf2, "bwd_ms": tb2, "fwd_tflops": fl / tf2 / 1e9, "bwd_tflops": 2.5 * fl / tb2 / 1e9,
                      "max_abs_vs_ours": float((of.float() - o.float()).abs().max())}
    except Exception as e:  # no sm_100 image in the wheel, etc.
        out["fa2"] = {"unavailable": repr(e)[:200]}
    try:
        import flashinfer
        wsb = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(wsb, "NHD")
        w.plan(cu, cu, H, Hkv, d, causal=causal, q_data_type=torch.bfloat16)
        tf3 = timed(lambda: w.run(q, k, v), a.iters)
        oi = w.run(q, k, v)
        out["flashinfer"] = {"fwd_ms": tf3, "fwd_tflops": fl / tf3 / 1e9,
                             "max_abs_vs_ours": float((oi.float() - o.float()).abs().max())}
    except Exception as e:
        out["flashinfer"] = {"unavailable": repr(e)[:200]}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
