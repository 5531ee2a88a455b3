"""The C ABI used from plain C (examples/certify.c): it compiles and links against include/polya.h and
libpolya.so with gcc here (no GPU needed), and on the GPU certifies its stable system and not the
unstable copy."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    import paper_1411_3769_b200 as pb
    pb.lib()   # make sure libpolya.so exists (and loads)
    libdir = os.path.join(ROOT, "paper_1411_3769_b200")
    out = str(tmp_path / "certify")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           os.path.join(ROOT, "examples", "certify.c"), "-L", libdir, "-lpolya", f"-Wl,-rpath,{libdir}",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_c_example_builds(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_example_certifies(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0].startswith("stable:") and lines[0].endswith("certified=1")
    assert lines[1].startswith("unstable:") and lines[1].endswith("certified=0")
