"""Attention-only timing for the parity configs (not the bench.py contract line).

  python tools/bench_attn.py --cfg 2|3|4 [--iters N]

cfg 2: GR00T-N1.5 shape (U[16,512] lengths, 8192-token bins, H16 d128, bidirectional) fwd + bwd.
cfg 3: pi0.5 shape (2 views x 256 + U[16,200] text + 50 action tokens; prefix = all but the 50
       action tokens), H8 d256 Hkv1 (MQA), prefix mask, fwd + bwd.
cfg 4: cfg-2 shape with E4M3 Q/K (per-block quantisation + the kind::f8f6f4 forward) vs bf16.
Kernel times by CUDA events on the launching stream after warm-up; inputs are packed once
(the packer is timed by bench.py).  TFLOP/s are algorithmic: 4·d·H per visible pair forward,
2.5x that backward.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11101_b200 import attention, fp8, packing, synthetic


def timed(fn, iters):
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(3):
        fn()
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
    ap.add_argument("--cfg", type=int, default=2, choices=[2, 3, 4])
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--samples", type=int, default=0)
    ap.add_argument("--seg-src", action="store_true", help="sample-major inputs through seg_src (as bench.py)")
    a = ap.parse_args()
    dev = torch.device("cuda")
    if a.cfg == 3:
        n = a.samples or 256
        L = synthetic.gen_lengths(n, synthetic.DIST_PI05, 16, 200, 50)
        H, Hkv, d, mask = 8, 1, 256, 2
    else:
        n = a.samples or 512
        L = synthetic.gen_lengths(n, synthetic.DIST_UNIFORM, 16, 512)
        H, Hkv, d, mask = 16, 16, 128, 0
    plan = packing.pack_ffd(L, 8192)
    T = plan.total_tokens()
    ids = plan.member_ids[:n].cpu().numpy()
    Lp = L[ids]  # segment order of the packed stream
    prefix_h = np.maximum(Lp - 50, 0).astype(np.int32) if mask == 2 else None
    prefix = torch.from_numpy(prefix_h).to(dev) if mask == 2 else None
    pairs = packing.visible_pairs(Lp.tolist(), mask, None if prefix_h is None else prefix_h.tolist())
    q = synthetic.fill_bf16(torch.empty(T, H, d, dtype=torch.bfloat16, device=dev), "q")
    k = synthetic.fill_bf16(torch.empty(T, Hkv, d, dtype=torch.bfloat16, device=dev), "k")
    v = synthetic.fill_bf16(torch.empty(T, Hkv, d, dtype=torch.bfloat16, device=dev), "v")
    do = synthetic.fill_bf16(torch.empty(T, H, d, dtype=torch.bfloat16, device=dev), "do")
    cu = plan.cu_seqlens[: n + 1]
    seg = packing.seg_src(plan) if a.seg_src else None
    o = torch.empty_like(q)
    lse = torch.empty(H, T, dtype=torch.float32, device=dev)
    ws = attention.BwdWorkspace()
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    fl = 4.0 * d * H * pairs
    out = {"cfg": a.cfg, "seg_src": a.seg_src, "samples": n, "tokens": T, "bins": plan.num_bins(), "H": H, "Hkv": Hkv, "d": d,
           "mask": mask, "pairs": pairs}

    def fwd():
        attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix, out=o, lse=lse, seg_src=seg)

    def bwd():
        attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, mask_mode=mask, prefix_len=prefix, workspace=ws,
                                  dq=dq, dk=dk, dv=dv, seg_src=seg)

    tf = timed(fwd, a.iters)
    out["fwd_ms"], out["fwd_tflops"] = tf, fl / tf / 1e9
    if a.cfg == 4:
        qc, qs = fp8.quant_block(q)
        kc, ks = fp8.quant_block(k)
        o8 = torch.empty_like(q)
        l8 = torch.empty_like(lse)

        def f8():
            fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, cu, out=o8, lse=l8, seg_src=seg)

        def quant():
            fp8.quant_block(q)
            fp8.quant_block(k)

        dq8, dk8, dv8 = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        ws8 = attention.BwdWorkspace()

        def b8():
            fp8.varlen_attn_bwd_fp8qk(do, qc, qs, kc, ks, v, o8, l8, cu, dq=dq8, dk=dk8, dv=dv8, seg_src=seg,
                                      workspace=ws8)

        t8 = timed(f8, a.iters)
        tq = timed(quant, a.iters)
        out["fp8_bwd_ms"] = timed(b8, a.iters)
        out["bwd_ms"] = timed(bwd, a.iters)
        out.update({"fp8_fwd_ms": t8, "fp8_fwd_tflops": fl / t8 / 1e9, "quant_qk_ms": tq,
                    "fp8_vs_bf16_max_abs": float((o8.float() - o.float()).abs().max())})
    else:
        tb = timed(bwd, a.iters)
        out["bwd_ms"], out["bwd_tflops"] = tb, 2.5 * fl / tb / 1e9
        out["fwd_bwd_tflops"] = 3.5 * fl / (tf + tb) / 1e9
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
