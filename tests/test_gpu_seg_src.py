"""Gather folded into the attention kernels (vlasim_attn_args.seg_src): attention over the
sample-major tensors with the packer's seg_src must equal, bit for bit, attention over the
explicitly gathered packed stream followed by the scatter back (SPEC.md:504 — the packed stream
is "concatenated tensors consistent with cu_seqlens"; here it is virtual)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = [
    # (n samples, max len, capacity, H, Hkv, d, mask)
    (40, 300, 1024, 2, 2, 128, 0),
    (40, 300, 1024, 4, 1, 128, 1),
    (60, 200, 512, 2, 2, 64, 0),
    (30, 400, 1024, 8, 1, 256, 2),
    (25, 260, 600, 2, 1, 256, 1),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_seg_src_matches_explicit_gather(gpu, case):
    from paper_2603_11101_b200 import attention, packing
    n, lmax, cap, H, Hkv, d, mask = CASES[case]
    rng = np.random.default_rng(case)
    L = rng.integers(1, lmax + 1, n).astype(np.int32)
    plan = packing.pack_ffd(L, cap)
    T = int(L.sum())
    g = torch.Generator(device="cuda").manual_seed(case)
    q, do = (torch.randn(T, H, d, device="cuda", generator=g).bfloat16() for _ in range(2))
    k, v = (torch.randn(T, Hkv, d, device="cuda", generator=g).bfloat16() for _ in range(2))
    cu = plan.cu_seqlens
    seg = packing.seg_src(plan)
    gidx = torch.empty(T, dtype=torch.int32, device="cuda")
    packing.token_ids_into(plan, T, gather_idx=gidx)
    Lp = np.diff(cu.cpu().numpy())
    prefix = torch.tensor(Lp // 3, dtype=torch.int32, device="cuda") if mask == 2 else None
    # explicit path: gather → attention on the packed stream → scatter back (row_map)
    qp, kp, vp, dop = (packing.gather_rows(x, plan) for x in (q, k, v, do))
    o_p, lse_p = attention.varlen_attn_fwd(qp, kp, vp, cu, mask_mode=mask, prefix_len=prefix)
    dq_p, dk_p, dv_p = attention.varlen_attn_bwd(dop, qp, kp, vp, o_p, lse_p, cu, mask_mode=mask,
                                                 prefix_len=prefix, row_map=gidx)
    # fused path: sample-major tensors + seg_src
    o_s, lse_s = attention.varlen_attn_fwd(q, k, v, cu, mask_mode=mask, prefix_len=prefix, seg_src=seg)
    dq_s, dk_s, dv_s = attention.varlen_attn_bwd(do, q, k, v, o_s, lse_s, cu, mask_mode=mask, prefix_len=prefix,
                                                 seg_src=seg)
    torch.cuda.synchronize()
    gl = gidx.long()
    assert torch.equal(o_s[gl], o_p)
    assert torch.equal(lse_s[:, gl], lse_p)
    assert torch.equal(dq_s, dq_p) and torch.equal(dk_s, dk_p) and torch.equal(dv_s, dv_p)


def test_seg_src_fp8_within_tolerance(gpu, orc):
    """FP8 Q/K forward on sample-major codes (scale blocks of source rows) vs the fp64 oracle."""
    from paper_2603_11101_b200 import fp8, packing
    rng = np.random.default_rng(9)
    L = rng.integers(1, 400, 30).astype(np.int32)
    plan = packing.pack_ffd(L, 1024)
    T, H, d = int(L.sum()), 2, 128
    g = torch.Generator(device="cuda").manual_seed(9)
    q, k, v = (torch.randn(T, H, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    qc, qs = fp8.quant_block(q)
    kc, ks = fp8.quant_block(k)
    o8, _ = fp8.varlen_attn_fwd_fp8qk(qc, qs, kc, ks, v, plan.cu_seqlens, seg_src=packing.seg_src(plan))
    gidx = torch.empty(T, dtype=torch.int32, device="cuda")
    packing.token_ids_into(plan, T, gather_idx=gidx)
    gl = gidx.long()
    f = lambda t: t.float().cpu().numpy()
    ro, _ = orc.mha_fwd(f(q[gl]), f(k[gl]), f(v[gl]), plan.cu_seqlens.cpu().numpy(), mask=0, prefix=None)
    err = np.max(np.abs(f(o8[gl]) - ro)) / max(1.0, np.max(np.abs(ro)))
    assert err < 6e-2, err


def test_seg_src_and_row_map_exclusive(gpu):
    from paper_2603_11101_b200 import attention, packing
    from paper_2603_11101_b200.errors import ConfigError
    L = np.array([5, 7], np.int32)
    plan = packing.pack_ffd(L, 16)
    q = torch.randn(12, 1, 64, device="cuda").bfloat16()
    seg = packing.seg_src(plan)
    o, lse = attention.varlen_attn_fwd(q, q, q, plan.cu_seqlens, seg_src=seg)
    with pytest.raises(ConfigError):
        attention.varlen_attn_bwd(q, q, q, q, o, lse, plan.cu_seqlens, seg_src=seg,
                                  row_map=torch.zeros(12, dtype=torch.int32, device="cuda"))


def test_sm_budget_is_bit_identical(gpu):
    """sm_budget only changes which CTA runs an item: outputs and gradients are bit-identical."""
    from paper_2603_11101_b200 import attention, packing
    rng = np.random.default_rng(3)
    L = rng.integers(1, 300, 40).astype(np.int32)
    plan = packing.pack_ffd(L, 1024)
    T, H, d = int(L.sum()), 4, 128
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v, do = (torch.randn(T, H, d, device="cuda", generator=g).bfloat16() for _ in range(4))
    seg = packing.seg_src(plan)
    cu = plan.cu_seqlens
    res = []
    for budget in (0, 7, 147):
        o, lse = attention.varlen_attn_fwd(q, k, v, cu, seg_src=seg, sm_budget=budget)
        grads = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, seg_src=seg, sm_budget=budget)
        res.append((o, lse) + tuple(grads))
    torch.cuda.synchronize()
    for other in res[1:]:
        assert all(torch.equal(x, y) for x, y in zip(res[0], other))


def test_config2_scale_consistency(gpu):
    """Race detector at the bench's scale (config 2: 512 samples U[16,512], 8192-token bins, H16
    d128, ~140 items per CTA): the fused layout must equal the explicit gather bit for bit (fwd and
    bwd), and the FP8 Q/K forward must stay within the FP8 tolerance of the bf16 one.  Pipelining
    bugs (stale barriers, early buffer reuse) only show once items queue up per CTA."""
    from paper_2603_11101_b200 import attention, fp8, packing, synthetic
    L = synthetic.gen_lengths(512, 0, 16, 512)
    plan = packing.pack_ffd(L, 8192)
    T, H, d = int(L.sum()), 16, 128
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v, do = (torch.randn(T, H, d, device="cuda", generator=g).bfloat16() for _ in range(4))
    cu, seg = plan.cu_seqlens, packing.seg_src(plan)
    gidx = torch.empty(T, dtype=torch.int32, device="cuda")
    packing.token_ids_into(plan, T, gather_idx=gidx)
    gl = gidx.long()
    o_s, lse_s = attention.varlen_attn_fwd(q, k, v, cu, seg_src=seg)
    dq_s, dk_s, dv_s = attention.varlen_attn_bwd(do, q, k, v, o_s, lse_s, cu, seg_src=seg)
    qp, kp, vp, dop = (x[gl].contiguous() for x in (q, k, v, do))
    o_p, lse_p = attention.varlen_attn_fwd(qp, kp, vp, cu)
    dq_p, dk_p, dv_p = attention.varlen_attn_bwd(dop, qp, kp, vp, o_p, lse_p, cu, row_map=gidx)
    qc, qsc = fp8.quant_block(q)
    kc, ksc = fp8.quant_block(k)
    o8, _ = fp8.varlen_attn_fwd_fp8qk(qc, qsc, kc, ksc, v, cu, seg_src=seg)
    torch.cuda.synchronize()
    assert torch.equal(o_s[gl], o_p) and torch.equal(lse_s[:, gl], lse_p)
    assert torch.equal(dq_s, dq_p) and torch.equal(dk_s, dk_p) and torch.equal(dv_s, dv_p)
    # north_star FP8 tolerance, relative to max(1, max|o|) (the bf16 output stands in for the reference)
    err = (o8.float() - o_s.float()).abs().max().item() / max(1.0, o_s.float().abs().max().item())
    assert err < 6e-2, err


_MODE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2603_11101_b200 import attention, packing, synthetic
L = synthetic.gen_lengths(96, 0, 16, 512)
plan = packing.pack_ffd(L, 4096)
T, H, d = int(L.sum()), 4, int(sys.argv[3])
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v, do = (torch.randn(T, H, d, device="cuda", generator=g).bfloat16() for _ in range(4))
cu, seg = plan.cu_seqlens, packing.seg_src(plan)
o, lse = attention.varlen_attn_fwd(q, k, v, cu, seg_src=seg)
dq, dk, dv = attention.varlen_attn_bwd(do, q, k, v, o, lse, cu, seg_src=seg)
np.savez(sys.argv[2], dk=dk.float().cpu().numpy(), dv=dv.float().cpu().numpy(), dq=dq.float().cpu().numpy())
"""


@pytest.mark.parametrize("d", [64, 128])
def test_dkdv_mode3_matches_mode0(gpu, tmp_path, d):
    """The default single-pass dK/dV kernel (K / V resident in TMEM, MODE 3) against the
    double-buffered one (VLASIM_DKV_MODE0): the same gradients (fresh processes: the switch is read
    once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for tag, env in (("m3", {}), ("m0", {"VLASIM_DKV_MODE0": "1"})):
        f = tmp_path / f"{tag}.npz"
        r = subprocess.run([sys.executable, "-c", _MODE_SCRIPT, root, str(f), str(d)],
                           env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[tag] = np.load(f)
    for key in ("dk", "dv", "dq"):
        a, b = outs["m3"][key], outs["m0"][key]
        assert np.allclose(a, b, rtol=0, atol=2e-2 * max(1.0, float(np.abs(b).max()))), key
