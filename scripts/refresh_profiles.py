"""Copy one gpu_final_r02.sh session (gpurun_out/*_TAG*) into profiles/r02/
with the ncu summaries (ncu_summary.py + ncu_lines.py) and the launch-list
summary.  Usage: python scripts/refresh_profiles.py TAG"""
import collections
import csv
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
g, p = ROOT / "gpurun_out", ROOT / "profiles" / "r02"
p.mkdir(parents=True, exist_ok=True)


def last(f):
    return (g / f).read_text().strip().splitlines()[-1] + "\n"


full = (g / f"bench_ref_{tag}.json").exists()   # gpu_final_r02.sh (else the short refresh)
(p / "bench.json").write_text(last(f"bench_{tag}.json"))
if full:
    (p / "bench_reference.json").write_text(last(f"bench_ref_{tag}.json"))
for src, dst in ((f"modes_{tag}.jsonl", "bench_modes.jsonl"), (f"configs_{tag}.jsonl", "configs.jsonl" if full else f"configs_{tag}.jsonl"),
                 (f"stats_{tag}.log", "kernel_stats.txt"), (f"pytest_{tag}.log", "pytest.log"),
                 (f"smoke_{tag}.log", "smoke.log"), (f"box_{tag}.txt", "box.txt"),
                 (f"sanitizer_{tag}.log", "sanitizer.log"), (f"launches_{tag}.csv", "launches.csv"),
                 (f"bricks_{tag}.jsonl", "bricks.jsonl"), (f"shard_{tag}.jsonl", "shard_timing.jsonl"),
                 (f"e2e_phases_{tag}.txt", "e2e_phases.txt"),
                 (f"pbuild_timing_{tag}.jsonl", "pbuild_timing.jsonl")):
    if (g / src).exists():
        shutil.copy(g / src, p / dst)
if (g / f"launches_{tag}.csv").exists():
    rows = [r for r in csv.reader(open(g / f"launches_{tag}.csv")) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split("(")[0].replace("<unnamed>::", "")[-48:]].append(float(r[vi].replace(",", "")))
    with open(p / "launches_summary.txt", "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, "
                f"bench.py --steps 3 --warmup 3 (radial272 skip-adaptive 512^2; {tag})\n")
        for k, v in d.items():
            f.write(f"{k:50s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.1f} us\n")


def summ(rep, out):
    if not rep.exists():
        return
    a = subprocess.run([sys.executable, str(ROOT / "scripts/ncu_summary.py"), str(rep)],
                       capture_output=True, text=True).stdout
    b = subprocess.run([sys.executable, str(ROOT / "scripts/ncu_lines.py"), str(rep), "30"],
                       capture_output=True, text=True).stdout
    (p / out).write_text(a + "\n# hottest source lines (all captured kernels)\n" + b)


summ(g / f"prof_march272_{tag}.ncu-rep", "ncu_march_kernel_radial272.txt")
summ(g / f"prof_trace272_{tag}.ncu-rep", "ncu_interval_kernels_radial272.txt")
summ(g / f"prof_march585_{tag}.ncu-rep", "ncu_march_kernel_grid585.txt")
print("profiles/r02 refreshed from", tag)
