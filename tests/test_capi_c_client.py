"""The C ABI from a plain C program (tools/capi_demo.c): no Python, no torch.

The CPU test compiles it against include/visloc_b200.h and the built library
(the ABI is plain C: structs, pointers, int status codes); the GPU test runs
it: 64 synthetic queries through one vl_ransac_pnp call on cudaMalloc'd
arrays, poses checked against the ground truth, vl_msac_score, and the
status codes of the reference's error cases (n < 3, bad config).
"""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2601_04185_b200" / "_lib"


def _compile(out):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None or not (LIB / "libvisloc_b200.so").exists():
        pytest.skip("no C compiler or library not built")
    cmd = [cc, "-O2", "-std=c11", str(ROOT / "tools" / "capi_demo.c"), f"-I{ROOT / 'include'}",
           "-I/usr/local/cuda/include", f"-L{LIB}", "-L/usr/local/cuda/lib64", "-lvisloc_b200", "-lcudart", "-lm",
           f"-Wl,-rpath,{LIB}", "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_client_compiles(tmp_path):
    _compile(tmp_path / "capi_demo")


@pytest.mark.gpu
def test_c_client_runs(tmp_path):
    exe = tmp_path / "capi_demo"
    _compile(exe)
    r = subprocess.run([str(exe), "64"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "converged 64" in r.stdout
