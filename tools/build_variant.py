"""Build an A/B variant of the library with extra -D flags for some sources.

    python tools/build_variant.py NAME "vl_ransac.cu:-DFOO -DBAR" ["vl_lift.cu:-DBAZ"]

Writes paper_2601_04185_b200/_lib/variant_NAME.so; select it at run time with
VISLOC_B200_LIB=<path> (tuning experiments only — the product build is
_build.py).
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_04185_b200._build import ARCH, COMMON, CSRC, NVCC, OUT_DIR, SOURCES, build  # noqa: E402


def main():
    name = sys.argv[1]
    extra = {}
    for spec in sys.argv[2:]:
        src, flags = spec.split(":", 1)
        extra[src] = flags.split()
    build()
    objs = []
    for s in SOURCES:
        o = OUT_DIR / s.replace(".cu", ".o")
        if s in extra:
            o = OUT_DIR / f"variant_{name}_{s.replace('.cu', '.o')}"
            subprocess.run([NVCC, *ARCH, *COMMON, *extra[s], "-c", str(CSRC / s), "-o", str(o)], check=True)
        objs.append(str(o))
    out = OUT_DIR / f"variant_{name}.so"
    subprocess.run([NVCC, *ARCH, "-shared", "-o", str(out), *objs, "-lcudart"], check=True)
    print(out)


if __name__ == "__main__":
    main()
