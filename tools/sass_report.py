"""ptxas resource usage and SASS instruction histograms of the library's kernels.

    python tools/sass_report.py > profiles/r02_sass_report.txt

Compiles every csrc/*.cu for sm_100a with -Xptxas -v (registers, spills,
shared memory per kernel) and histograms the SASS of the built objects
(cuobjdump -sass): the mnemonics that show the design — FFMA2/FMUL2 (packed
FP32) and MUFU.RCP in k_score, UBLKCP (cp.async.bulk, TMA) + SYNCS (mbarrier)
in the LM / MSAC / lift kernels, DFMA/DMUL in the fp64 kernels.
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2601_04185_b200" / "csrc"
sys.path.insert(0, str(ROOT))
from paper_2601_04185_b200._build import ARCH, COMMON, NVCC, OUT_DIR, SOURCES  # noqa: E402

KEY = ("FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "MUFU", "FMNMX", "DFMA", "DMUL", "DADD", "LDS", "STS", "LDG",
       "STG", "LDL", "STL", "UBLKCP", "SYNCS", "SHFL", "BAR", "REDUX")


def main():
    print("# ptxas -v (sm_100a)\n")
    for src in SOURCES:
        r = subprocess.run([NVCC, *ARCH, *COMMON, "-c", str(CSRC / src), "-o", "/dev/null", "-Xptxas", "-v"],
                           capture_output=True, text=True)
        fn, spill = None, ""
        for ln in r.stderr.splitlines():
            m = re.search(r"Compiling entry function '(\S+)'", ln)
            if m:
                fn, spill = m.group(1), ""
                continue
            m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
            if m and fn:  # ptxas prints the frame line before the register line
                spill = f"  stack {m.group(1)} B, spill st {m.group(2)} / ld {m.group(3)} B"
                continue
            m = re.search(r"Used (\d+) registers", ln)
            if m and fn:
                sm = re.search(r"(\d+) bytes smem", ln)
                dem = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
                print(f"{src:16s} {dem[:80]:80s} regs {m.group(1):>4s} smem {sm.group(1) if sm else '0':>6s}{spill}")
                fn = None
    print("\n# SASS instruction histograms (static counts per kernel, selected mnemonics)\n")
    for src in SOURCES:
        obj = OUT_DIR / (Path(src).stem + ".o")
        sass = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True).stdout
        for block in re.split(r"\n\s+Function : ", sass)[1:]:
            name = block.split("\n", 1)[0].strip()
            ops = collections.Counter()
            for ln in block.splitlines():
                m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", ln)
                if m:
                    ops[m.group(1)] += 1
            total = sum(ops.values())
            if total < 50:
                continue
            dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            sel = ", ".join(f"{k} {ops[k]}" for k in KEY if ops[k])
            print(f"{dem[:100]}\n    {total} instructions: {sel}")


if __name__ == "__main__":
    main()
