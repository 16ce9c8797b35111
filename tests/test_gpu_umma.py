"""tcgen05 / TMA / TMEM layout self-test: the single-CTA UMMA GEMM used to validate every operand
layout the attention kernels rely on, against a torch fp32 matmul."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(mode, a, b, N):
    from paper_2603_11101_b200 import _lib
    c = torch.empty(128, N, dtype=torch.float32, device="cuda")
    K = a.shape[1] if mode != 3 else a.shape[0]
    _lib.check(_lib.lib().vlasim_selftest_umma(mode, _lib.ptr(a), _lib.ptr(b), _lib.ptr(c, _lib.f32p), N, K,
                                               _lib.stream_ptr()), "selftest")
    torch.cuda.synchronize()
    return c


@pytest.mark.parametrize("N,K", [(128, 128), (64, 64), (256, 128), (128, 256), (64, 256)])
@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
def test_umma_layouts(gpu, mode, N, K):
    g = torch.Generator(device="cuda").manual_seed(mode * 1000 + N + K)
    if mode == 3:
        a = torch.randn(K, 128, device="cuda", generator=g).bfloat16()
    else:
        a = torch.randn(128, K, device="cuda", generator=g).bfloat16()
    if mode == 0:
        b = torch.randn(N, K, device="cuda", generator=g).bfloat16()
        ref = a.float() @ b.float().t()
    else:
        b = torch.randn(K, N, device="cuda", generator=g).bfloat16()
        ref = (a.float().t() if mode == 3 else a.float()) @ b.float()
    c = _run(mode, a, b, N)
    err = (c - ref).abs().max().item()
    assert err < 1e-3 * max(1.0, ref.abs().max().item()), f"mode {mode} N {N} K {K}: max err {err}"
