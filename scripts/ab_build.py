"""Build A/B variants of libtetray_b200.so with extra -D macros into
build/ab/<name>/libtetray_b200.so (select one with TETRAY_B200_LIB=...).

    python scripts/ab_build.py name=-DTR_FIELD_PREFETCH=0 [name2=-DX=1,-DY=2 ...]
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1908_01906_b200 import _build as Bd  # noqa: E402

for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    out = ROOT / "build" / "ab" / name / "libtetray_b200.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    Bd.build_library()   # also refreshes the generated glibc pow header
    cmd = [Bd._nvcc(), *Bd.NVCC_FLAGS, *[d for d in defs.split(",") if d], "-ccbin", "/usr/bin/g++",
           "-I", str(ROOT / "include"), "-I", str(Bd.CSRC),
           *[str(Bd.CSRC / s) for s in Bd.SOURCES], "-o", str(out), "-lgomp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode:
        sys.exit(res.stderr[-3000:])
    print(out)
