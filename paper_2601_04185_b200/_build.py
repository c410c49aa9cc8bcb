"""Build the sm_100a shared library (libvisloc_b200.so) in-tree with nvcc.

The library is the product: every hot-path entry point of the Python package
binds to it through ctypes (see ``_lib.py``).  Built for sm_100a only — no
PTX fallback, no other architectures.
"""

from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
OUT_DIR = HERE / "_lib"
LIB = OUT_DIR / "libvisloc_b200.so"
HOSTCHECK = OUT_DIR / "libvisloc_hostcheck.so"
SOURCES = ["vl_capi.cu", "vl_ransac.cu", "vl_score.cu", "vl_lift.cu", "vl_imlc.cu", "vl_retrieval.cu", "vl_mapcodec.cu", "vl_tri.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", str(HERE.parent / "include")]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + \
        list((HERE.parent / "include").glob("*.h"))
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_v: bool = False) -> Path:
    OUT_DIR.mkdir(exist_ok=True)
    objs = []
    jobs = []
    for s in SOURCES:
        src = CSRC / s
        obj = OUT_DIR / (Path(s).stem + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            cmd = [NVCC, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
            if ptxas_v:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stdout + r.stderr

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        for out in ex.map(run, jobs):
            if verbose and out.strip():
                print(out)
    if force or jobs or not LIB.exists():
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
        run(cmd)
    hsrc = CSRC / "vl_hostcheck.cu"
    if force or _stale(HOSTCHECK, hsrc):
        # host-only build of the __host__ __device__ solver cores (CPU unit tests)
        run([NVCC, *COMMON, "-shared", "-o", str(HOSTCHECK), str(hsrc)])
    return LIB


if __name__ == "__main__":
    import sys
    print(build(verbose=True, force="--force" in sys.argv, ptxas_v="-v" in sys.argv))
