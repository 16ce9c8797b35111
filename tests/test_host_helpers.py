"""the SPEC's scalar helpers exist as the C++ drop-in (libvlasim.so), the Python
mirror (paper_2603_11101_b200) and the oracle — held to the same values here, on the SPEC's examples
and random cases (CPU only; the C++ copy runs through tests/dropin/host_helpers.cpp)."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2603_11101_b200" / "lib"
CUDA = Path("/usr/local/cuda")


@pytest.fixture(scope="module")
def cpp(tmp_path_factory):
    exe = tmp_path_factory.mktemp("hh") / "host_helpers"
    cmd = ["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
           str(ROOT / "tests" / "dropin" / "host_helpers.cpp"), "-o", str(exe), "-L", str(LIB), "-lvlasim",
           "-lvlasim_cuda", f"-Wl,-rpath,{LIB}", "-L", str(CUDA / "lib64"), "-lcudart", f"-Wl,-rpath,{CUDA / 'lib64'}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

    def run(lines):
        r = subprocess.run([str(exe)], input="\n".join(lines) + "\n", capture_output=True, text=True, timeout=60)
        assert r.returncode == 0, r.stderr
        return [json.loads(x) for x in r.stdout.strip().splitlines()]
    return run


def _cases():
    rng = np.random.default_rng(0)
    cases = [([10, 5, 5], 10, 64), ([37, 120, 85], 120, 128), ([64] * 5, 64, 16), ([8192, 4096], 8192, 128)]
    for _ in range(40):
        L = rng.integers(1, 3000, int(rng.integers(1, 60))).tolist()
        cases.append((L, max(L) + int(rng.integers(0, 500)), int(rng.choice([16, 64, 128, 256]))))
    return cases


def test_lengths_helpers_three_copies_agree(cpp):
    from oracle import oracle as orc
    from paper_2603_11101_b200 import packing
    cases = _cases()
    out = cpp([f"lengths {p} {d} " + " ".join(map(str, L)) for L, p, d in cases])
    for (L, p, d), c in zip(cases, out):
        assert c["padding_rate"] == packing.padding_rate(L, p) == pytest.approx(orc.padding_rate(L, p), abs=0)
        assert c["dynamic_pad_length"] == packing.dynamic_pad_length(L) == orc.dynamic_pad_length(L)
        assert c["flops_fixed"] == packing.attention_flops(L, d, p) == orc.attention_flops(L, d, p)
        assert c["flops_packed"] == packing.attention_flops(L, d) == orc.attention_flops(L, d)
    assert out[0]["padding_rate"] == pytest.approx(1 / 3)
    assert out[1]["dynamic_pad_length"] == 120


def test_packing_stats_against_oracle(cpp):
    from oracle import oracle as orc
    rng = np.random.default_rng(1)
    lines, expect = [], []
    for _ in range(20):
        L = rng.integers(16, 513, 64)
        bin_of, slot, tok, nb = orc.pack(L, 2048, 0)
        bins = [[int(L[i]) for i in sorted(np.flatnonzero(bin_of == b), key=lambda i: slot[i])] for b in range(nb)]
        pad = int(L.max())
        lines.append(f"stats 2048 {pad} 64 {nb} " + " ".join(f"{len(m)} " + " ".join(map(str, m)) for m in bins))
        expect.append((L, nb, pad))
    for (L, nb, pad), c in zip(expect, cpp(lines)):
        assert c["bins_used"] == nb
        assert c["fill_rate"] == pytest.approx(L.sum() / (nb * 2048), rel=1e-15)
        assert c["padding_rate_after"] == pytest.approx(1 - L.sum() / (nb * 2048), rel=1e-12)
        assert c["padding_rate_before"] == orc.padding_rate(L.tolist(), pad)
        assert c["flops_packed"] == orc.attention_flops(L.tolist(), 64)
        assert c["flops_packed"] <= c["flops_fixed"]


def test_quant_and_prune_helpers_agree(cpp):
    from paper_2603_11101_b200 import quant
    from paper_2603_11101_b200.packing import SampleLen, prune_view
    shapes = [(256, 256), (200, 300), (1, 1), (129, 4097)]
    out = cpp([f"blocks {r} {c}" for r, c in shapes])
    for (r, c), o in zip(shapes, out):
        assert o["blocks"] == len(quant.block_partition((r, c))) and o["area"] == r * c
    assert [o["blocks"] for o in out[:2]] == [4, 6]
    comp = cpp(["compression 2 1 0 1000000000 q 100000000 q", "compression 2 1 4 1000 k",
                "compression 2 1 4 668684288 k 311164928 k 241664 k 2774532096 q"])
    assert comp[0]["compression_ratio"] == pytest.approx(0.5)
    assert comp[1]["compression_ratio"] == 0.0
    spec = quant.ModelSizeSpec([quant.ModelComponent("a", 668684288, False), quant.ModelComponent("b", 311164928, False),
                                quant.ModelComponent("c", 241664, False), quant.ModelComponent("d", 2774532096, True)])
    assert comp[2]["compression_ratio"] == pytest.approx(quant.compression_ratio(spec), rel=1e-15)
    pr = cpp(["prune 48 left=256 right=256 -- right", "prune 48 left=256 -- right"])
    assert pr[0]["total_len"] == 304 == prune_view(SampleLen(0, {"left": 256, "right": 256}, 48), "right").total_len
    assert "config_error" in pr[1]
