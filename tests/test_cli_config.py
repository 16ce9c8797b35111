"""Strict-schema configs and the `pack` / `quantbench` CLIs: unknown keys rejected
naming the key (exit 2), deterministic output files, the quantbench tables against the GPU quantizer
and the oracle."""
import json
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
PACK = ROOT / "paper_2603_11101_b200/lib/vlasim_pack"
QB = ROOT / "paper_2603_11101_b200/lib/vlasim_quantbench"
GOLDEN = ROOT / "tests/golden"


def run(*args):
    return subprocess.run([str(a) for a in args], capture_output=True, text=True)


def write_vlt(path, x):
    x = np.ascontiguousarray(x, np.float64)
    with open(path, "wb") as f:
        f.write(b"VLT1" + struct.pack("<I", x.ndim) + struct.pack(f"<{x.ndim}q", *x.shape) + x.tobytes())


def test_pack_config_unknown_key_is_named(tmp_path):  # SPEC.md:652-654 ("b_maxx")
    cfg = tmp_path / "run.cfg"
    cfg.write_text("seed = 7\n[packing]\ncapacity = 2048\nb_maxx = 3\n[synthetic]\nn = 64\n")
    r = run(PACK, "--config", cfg)
    assert r.returncode == 2 and "b_maxx" in r.stderr and ":4:" in r.stderr


@pytest.mark.parametrize("body,needle", [("[packing\ncapacity = 8\n", "section"),
                                         ("capacity 8\n", "key = value"),
                                         ("[packing]\ncapacity = 8\ncapacity = 9\n", "duplicate"),
                                         ("[packing]\ncapacity = eight\n", "integer"),
                                         ("[packing]\ncapacity = 8\nalgorithm = best\n[synthetic]\nn = 3\n", "ffd or greedy")])
def test_pack_config_malformed(tmp_path, body, needle):
    cfg = tmp_path / "bad.cfg"
    cfg.write_text(body)
    r = run(PACK, "--config", cfg)
    assert r.returncode == 2 and needle in r.stderr, r.stderr


def test_pack_prune_missing_view_is_error(tmp_path):  # unknown view → error
    f = tmp_path / "corpus.txt"
    f.write_text("0 48 left=256 right=256\n1 30 left=256\n")
    r = run(PACK, "--capacity", "4096", "--corpus", f, "--prune", "right")
    assert r.returncode == 2 and "right" in r.stderr


def test_quantbench_config_unknown_key(tmp_path):
    cfg = tmp_path / "q.cfg"
    cfg.write_text("[quantization]\ngranularities = block\ngranularitys = tensor\n")
    r = run(QB, "--config", cfg)
    assert r.returncode == 2 and "granularitys" in r.stderr


def test_quantbench_non_finite_fixture(tmp_path):  # non-finite fixture values → error
    x = np.ones((4, 4))
    x[1, 2] = np.nan
    write_vlt(tmp_path / "bad.vlt", x)
    r = run(QB, "--fixture", tmp_path / "bad.vlt", "--granularity", "tensor")
    assert r.returncode == 2 and "non-finite" in r.stderr


@pytest.mark.gpu
def test_pack_config_run_is_deterministic(gpu, orc, tmp_path):
    rng = np.random.default_rng(9)
    L = rng.integers(260, 900, 200).tolist()
    (tmp_path / "corpus.txt").write_text("\n".join(f"{i} {l - 256} left=256" for i, l in enumerate(L)) + "\n")
    cfg = tmp_path / "run.cfg"
    cfg.write_text(f"seed = 1\nout = {tmp_path}/o1\n[packing]\ncorpus = {tmp_path}/corpus.txt\ncapacity = 2048\n"
                   "algorithm = ffd\nmanifest = no\n")
    assert run(PACK, "--config", cfg).returncode == 0
    assert run(PACK, "--config", cfg, "--out", tmp_path / "o2").returncode == 0
    for f in ("stats.json", "manifest.tsv"):
        assert (tmp_path / "o1" / f).read_bytes() == (tmp_path / "o2" / f).read_bytes()
    stats = json.loads((tmp_path / "o1/stats.json").read_text())
    bin_of, slot, tok, nb = orc.pack(L, 2048, 0)
    assert stats["bins_used"] == nb
    rows = (tmp_path / "o1/manifest.tsv").read_text().splitlines()
    assert len(rows) == nb
    for line in rows:
        parts = line.split()
        mem = [int(x) for x in parts[parts.index("members") + 1: parts.index("cu_seqlens")]]
        assert all(bin_of[i] == int(parts[1]) for i in mem)


@pytest.mark.gpu
def test_quantbench_tables(gpu, orc, tmp_path):
    rng = np.random.default_rng(1)
    x = (rng.standard_normal((300, 260)) * rng.choice([0.01, 1.0, 50.0], (300, 1))).astype(np.float32)
    write_vlt(tmp_path / "w.vlt", x)
    (tmp_path / "w.txt").write_text("# small text fixture\n2 3\n1 -2 3.5\n0 448 -448\n")
    p = json.loads((GOLDEN / "qwen25vl_3b_params.json").read_text())
    spec = tmp_path / "model.cfg"
    spec.write_text(f"component.vision = {p['vision']} keep\ncomponent.embeddings = {p['embeddings']} keep\n"
                    f"component.lm_1d = {p['lm_1d']} keep\ncomponent.lm_linear = {p['lm_linear']} quantize block\n")
    r = run(QB, "--fixture", tmp_path / "w.vlt", "--fixture", tmp_path / "w.txt", "--granularity",
            "tensor,channel:0,channel:1,block", "--model-spec", spec, "--out", tmp_path / "out")
    assert r.returncode == 0, r.stderr
    lines = (tmp_path / "out/quantbench.tsv").read_text().strip().splitlines()
    assert lines[0].split("\t")[:3] == ["fixture", "granularity", "groups"]
    rows = {(l.split("\t")[0], l.split("\t")[1]): l.split("\t") for l in lines[1:]}
    for g, axis, name in (("tensor", 0, "tensor"), ("channel", 0, "channel:0"), ("channel", 1, "channel:1"),
                          ("block", 0, "block")):
        codes, scales = orc.fp8_quantize(x, g, axis)
        _, _, _, mx, mse = orc.fp8_quant_error_general(x, codes, scales, g, axis)
        row = rows[(str(tmp_path / "w.vlt"), name)]
        assert int(row[2]) == scales.size
        assert float(row[3]) == pytest.approx(mx, rel=1e-8)
        assert float(row[4]) == pytest.approx(mse, rel=1e-8)
    small = rows[(str(tmp_path / "w.txt"), "tensor")]
    assert float(small[3]) == 0.0 and float(small[4]) == 0.0  # values exact at scale 1
    comp = (tmp_path / "out/compression.tsv").read_text().strip().splitlines()
    ratio = float(comp[-1].split("\t")[1])
    assert abs(ratio - 0.366) <= 0.01
