"""Oracle parity at the BENCHMARKED configurations, at their full scale (BASELINE.json configs[0..3]).

The inputs are exactly bench.py's: lengths from make_rng(42, "lengths", 0) (rng.hpp), GPU FFD packing,
sample-major counter-based synthetic Q/K/V/dO (labels "q", "k", "v", "do", root 42) read through
seg_src — the fused layout the bench step times.  Every packed segment runs through the persistent
schedulers, cost-bucket sort and tile tables at the real item counts; the fp64 oracle
(oracle/vlasim_oracle.cpp, SPEC.md:502-509 + the closed-form backward) then checks

  config 2  (512 × U[16,512], 8192-token bins, H16 d128, bidirectional):  O, LSE, dQ, dK, dV of heads
            {0, 15} over EVERY segment (MHA: head h's dK/dV depend on head h only);
  config 1  (64 × U[16,512], 2048-token bins, H8 d64): all heads, all segments;
  config 3  (π0.5: 512 + U[16,200] + 50 tokens, prefix = all but the 50 action tokens, H8 Hkv1 d256,
            prefix mask): O / LSE / dQ of heads {0, 7} over every segment; dK / dV (a sum over all
            8 query heads under MQA) over every 8th segment with all heads;
  config 4  (config 2 with E4M3 Q/K): O of heads {0, 15} over every segment vs the fp64 oracle on the
            original bf16 inputs, and the FP8 backward's gradients.

Tolerances are north_star's: max |gpu − ref| ≤ 2e-2 · max(1, max|ref|) for bf16, 6e-2 for FP8.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL_BF16, TOL_FP8 = 2e-2, 6e-2


def _err(x, ref):
    x = np.asarray(x, np.float64)
    return float(np.max(np.abs(x - ref)) / max(1.0, np.max(np.abs(ref))))


def _setup(n, dist, p, cap, H, Hkv, d):
    from paper_2603_11101_b200 import packing, synthetic
    L = synthetic.gen_lengths(n, dist, *p)
    plan = packing.pack_ffd(L, cap)
    T = int(L.sum())
    dev = torch.device("cuda")
    q = synthetic.fill_bf16(torch.empty(T, H, d, dtype=torch.bfloat16, device=dev), "q")
    k = synthetic.fill_bf16(torch.empty(T, Hkv, d, dtype=torch.bfloat16, device=dev), "k")
    v = synthetic.fill_bf16(torch.empty(T, Hkv, d, dtype=torch.bfloat16, device=dev), "v")
    do = synthetic.fill_bf16(torch.empty(T, H, d, dtype=torch.bfloat16, device=dev), "do")
    seg = packing.seg_src(plan)
    gidx = torch.empty(T, dtype=torch.int32, device=dev)
    packing.token_ids_into(plan, T, gather_idx=gidx)
    return L, plan, (q, k, v, do), seg, gidx.long()


def _check_plan(orc, L, plan, cap):
    bin_of, slot, tok, nb = orc.pack(L, cap, 0)
    assert plan.num_bins() == nb
    assert np.array_equal(plan.bin_of.cpu().numpy(), bin_of)
    assert np.array_equal(plan.slot.cpu().numpy(), slot)


def _packed(x, gl, heads=None):
    """Packed-stream rows (fp64 host) of a sample-major tensor, optionally a subset of heads."""
    y = x[gl]
    if heads is not None:
        y = y[:, heads]
    return y.float().cpu().numpy().astype(np.float64)


def _subset(cu, segs, *arrays):
    """Rows of the packed segments `segs` as a compact packed stream with its own cu_seqlens."""
    idx = np.concatenate([np.arange(cu[s], cu[s + 1]) for s in segs])
    lens = np.array([cu[s + 1] - cu[s] for s in segs])
    cu2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    return cu2, idx, [a[idx] for a in arrays]


def _run_bf16(qkvdo, cu, seg, mask=0, prefix=None):
    from paper_2603_11101_b200 import attention
    q, k, v, do = qkvdo
    o, lse = attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix, seg_src=seg)
    dq, dk, dv = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, mask_mode=mask, prefix_len=prefix, seg_src=seg)
    torch.cuda.synchronize()
    return o, lse, dq, dk, dv


def test_config2_full_scale_vs_oracle(gpu, orc):
    from paper_2603_11101_b200 import synthetic
    H, d = 16, 128
    L, plan, qkvdo, seg, gl = _setup(512, synthetic.DIST_UNIFORM, (16, 512), 8192, H, H, d)
    _check_plan(orc, L, plan, 8192)
    assert plan.num_bins() == 17
    cu_d = plan.cu_seqlens
    o, lse, dq, dk, dv = _run_bf16(qkvdo, cu_d, seg)
    cu = cu_d.cpu().numpy()
    heads = [0, H - 1]
    q, k, v, do = (_packed(x, gl, heads) for x in qkvdo)
    ro, rlse = orc.mha_fwd(q, k, v, cu)
    rdq, rdk, rdv = orc.mha_bwd(q, k, v, ro, do, cu)
    assert _err(_packed(o, gl, heads), ro) < TOL_BF16, "o"
    lse_p = lse[:, gl][heads].cpu().numpy()
    assert np.max(np.abs(lse_p - rlse)) < 1e-2, "lse"
    assert _err(_packed(dv, gl, heads), rdv) < TOL_BF16, "dv"
    assert _err(_packed(dk, gl, heads), rdk) < TOL_BF16, "dk"
    assert _err(_packed(dq, gl, heads), rdq) < TOL_BF16, "dq"


def test_config1_full_vs_oracle(gpu, orc):
    from paper_2603_11101_b200 import synthetic
    H, d = 8, 64
    L, plan, qkvdo, seg, gl = _setup(64, synthetic.DIST_UNIFORM, (16, 512), 2048, H, H, d)
    _check_plan(orc, L, plan, 2048)
    assert plan.num_bins() == 8 and int(L.sum()) == 15117
    o, lse, dq, dk, dv = _run_bf16(qkvdo, plan.cu_seqlens, seg)
    cu = plan.cu_seqlens.cpu().numpy()
    q, k, v, do = (_packed(x, gl) for x in qkvdo)
    ro, rlse = orc.mha_fwd(q, k, v, cu)
    rdq, rdk, rdv = orc.mha_bwd(q, k, v, ro, do, cu)
    assert _err(_packed(o, gl), ro) < TOL_BF16
    assert np.max(np.abs(lse[:, gl].cpu().numpy() - rlse)) < 1e-2
    for name, x, r in (("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        assert _err(_packed(x, gl), r) < TOL_BF16, name
    # config 1 as BASELINE states it (fp32 forward): the oracle's fp32 path agrees with fp64 too
    ro32, _ = orc.mha_fwd(q, k, v, cu, dtype=np.float32)
    assert _err(ro32, ro) < 1e-4


def test_config3_full_scale_vs_oracle(gpu, orc):
    from paper_2603_11101_b200 import synthetic
    H, Hkv, d = 8, 1, 256
    L, plan, qkvdo, seg, gl = _setup(256, synthetic.DIST_PI05, (16, 200, 50), 8192, H, Hkv, d)
    _check_plan(orc, L, plan, 8192)
    n = L.size
    Lp = L[plan.member_ids[:n].cpu().numpy()]  # segment (packed) order
    prefix = torch.tensor(Lp - 50, dtype=torch.int32, device="cuda")
    o, lse, dq, dk, dv = _run_bf16(qkvdo, plan.cu_seqlens, seg, mask=2, prefix=prefix)
    cu = plan.cu_seqlens.cpu().numpy()
    pre = prefix.cpu().numpy()
    heads = [0, H - 1]
    q2, do2 = _packed(qkvdo[0], gl, heads), _packed(qkvdo[3], gl, heads)
    k, v = _packed(qkvdo[1], gl), _packed(qkvdo[2], gl)
    ro, rlse = orc.mha_fwd(q2, k, v, cu, mask=2, prefix=pre)
    assert _err(_packed(o, gl, heads), ro) < TOL_BF16, "o"
    assert np.max(np.abs(lse[:, gl][heads].cpu().numpy() - rlse)) < 1e-2, "lse"
    rdq, _, _ = orc.mha_bwd(q2, k, v, ro, do2, cu, mask=2, prefix=pre)
    assert _err(_packed(dq, gl, heads), rdq) < TOL_BF16, "dq"
    # dK / dV sum over all 8 query heads (MQA): every 8th segment, all heads
    segs = list(range(0, n, 8))
    qa, doa = _packed(qkvdo[0], gl), _packed(qkvdo[3], gl)
    cu2, idx, (qs, ks, vs, dos) = _subset(cu, segs, qa, k, v, doa)
    ro_s, _ = orc.mha_fwd(qs, ks, vs, cu2, mask=2, prefix=pre[segs])
    _, rdk, rdv = orc.mha_bwd(qs, ks, vs, ro_s, dos, cu2, mask=2, prefix=pre[segs])
    assert _err(_packed(dk, gl)[idx], rdk) < TOL_BF16, "dk"
    assert _err(_packed(dv, gl)[idx], rdv) < TOL_BF16, "dv"


def test_config4_fp8_full_scale_vs_oracle(gpu, orc):
    from paper_2603_11101_b200 import fp8, synthetic
    H, d = 16, 128
    L, plan, qkvdo, seg, gl = _setup(512, synthetic.DIST_UNIFORM, (16, 512), 8192, H, H, d)
    q, k, v, do = qkvdo
    cu_d = plan.cu_seqlens
    qc, qs = fp8.quant_block(q)
    kc, ks = fp8.quant_block(k)
    o8, lse8 = fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, cu_d, seg_src=seg)
    dq8, dk8, dv8 = fp8.varlen_attn_bwd_fp8qk(do, qc, qs, kc, ks, v, o8, lse8, cu_d, seg_src=seg)
    torch.cuda.synchronize()
    cu = cu_d.cpu().numpy()
    heads = [0, H - 1]
    qh, kh, vh, doh = (_packed(x, gl, heads) for x in qkvdo)
    ro, _ = orc.mha_fwd(qh, kh, vh, cu)
    rdq, rdk, rdv = orc.mha_bwd(qh, kh, vh, ro, doh, cu)
    assert _err(_packed(o8, gl, heads), ro) < TOL_FP8, "o"
    for name, x, r in (("dq", dq8, rdq), ("dk", dk8, rdk), ("dv", dv8, rdv)):
        assert _err(_packed(x, gl, heads), r) < TOL_FP8, name
