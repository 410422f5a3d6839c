"""Build A/B variants of libtetray_b200.so with extra -D macros into
build/ab/<name>/libtetray_b200.so (select one with TETRAY_B200_LIB=...).

    python scripts/ab_build.py name=-DTR_FIELD_PREFETCH=0 [name2=-DX=1,-DY=2 ...]
    python scripts/ab_build.py head=@HEAD        # the committed sources of a git revision
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
    csrc, inc = Bd.CSRC, ROOT / "include"
    if defs.startswith("@"):   # sources of a git revision, into a scratch tree
        rev, defs = defs[1:], ""
        tmp = Path("/tmp/ab_src") / name
        (tmp / "csrc").mkdir(parents=True, exist_ok=True)
        (tmp / "include").mkdir(parents=True, exist_ok=True)
        listing = subprocess.run(["git", "-C", str(ROOT), "ls-tree", "--name-only", rev,
                                  "paper_1908_01906_b200/csrc/"], capture_output=True, text=True,
                                 check=True).stdout.split()
        for path in listing:   # every source and header of that revision
            (tmp / "csrc" / Path(path).name).write_bytes(subprocess.run(
                ["git", "-C", str(ROOT), "show", f"{rev}:{path}"], capture_output=True,
                check=True).stdout)
        (tmp / "include" / "tetray_b200.h").write_bytes(subprocess.run(
            ["git", "-C", str(ROOT), "show", f"{rev}:include/tetray_b200.h"],
            capture_output=True, check=True).stdout)
        (tmp / "csrc" / "glibc_pow_data.h").write_bytes((Bd.CSRC / "glibc_pow_data.h").read_bytes())
        csrc, inc = tmp / "csrc", tmp / "include"
    cmd = [Bd._nvcc(), *Bd.NVCC_FLAGS, *[d for d in defs.split(",") if d], "-ccbin", "/usr/bin/g++",
           "-I", str(inc), "-I", str(csrc),
           *[str(csrc / s) for s in Bd.SOURCES], "-o", str(out), "-lgomp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode:
        sys.exit(res.stderr[-3000:])
    print(out)
