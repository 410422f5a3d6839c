"""Build A/B variants of libtetray_b200.so into build/ab/lib_<name>.so.

Each variant is the current csrc with a list of (old, new) text edits applied
to render.cu.  Usage: python scripts/ab_build.py  (edit VARIANTS below)."""
import shutil, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1908_01906_b200 import _build

VARIANTS = {
    "cur": [],
    "iv32": [("constexpr int IV_CAP = 64;", "constexpr int IV_CAP = 32;")],
    "iv16": [("constexpr int IV_CAP = 64;", "constexpr int IV_CAP = 16;")],
    "iv8": [("constexpr int IV_CAP = 64;", "constexpr int IV_CAP = 8;")],
}

def build(name, edits):
    d = ROOT / "build" / "ab" / name
    if d.exists():
        shutil.rmtree(d)
    shutil.copytree(_build.CSRC, d)
    if isinstance(edits, str) and edits.startswith("git:"):
        src = subprocess.run(["git", "show", edits[4:] + ":paper_1908_01906_b200/csrc/render.cu"],
                             capture_output=True, text=True, cwd=ROOT, check=True).stdout
        edits = []
    else:
        src = (d / "render.cu").read_text()
    for old, new in edits:
        assert old in src, (name, old)
        src = src.replace(old, new)
    (d / "render.cu").write_text(src)
    out = ROOT / "build" / "ab" / f"lib_{name}.so"
    cmd = [_build._nvcc(), *_build.NVCC_FLAGS, "-ccbin", "/usr/bin/g++", "-I", str(ROOT / "include"),
           "-I", str(d), *[str(d / s) for s in _build.SOURCES], "-o", str(out), "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-3000:]); raise SystemExit(1)
    print("built", out)

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        build(n, VARIANTS[n])
