"""The reconstructed vlasim:: C++ drop-in (libvlasim.so) called from C++ the way the reference's own
tests would call it: tests/dropin/test_dropin.cpp runs the SPEC's known-answer examples for
reference_attention / packed_attention, the 200-instance acceptance check
(lengths <= 64, dim <= 16), every model_dim class boundary 1..256, and pack_ffd /
cu_seqlens / error cases."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2603_11101_b200" / "lib"
CUDA = Path("/usr/local/cuda")


def _build(tmp_path):
    exe = tmp_path / "test_dropin"
    cmd = ["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
           str(ROOT / "tests" / "dropin" / "test_dropin.cpp"), "-o", str(exe), "-L", str(LIB), "-lvlasim",
           "-lvlasim_cuda", f"-Wl,-rpath,{LIB}", "-L", str(CUDA / "lib64"), "-lcudart", f"-Wl,-rpath,{CUDA / 'lib64'}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_dropin_cpp_builds_and_links(tmp_path):
    assert (LIB / "libvlasim.so").exists()
    _build(tmp_path)


@pytest.mark.gpu
def test_dropin_cpp_spec_known_answers(gpu, tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all SPEC known-answer checks passed" in r.stdout
