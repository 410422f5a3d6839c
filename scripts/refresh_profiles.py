"""Copy one gpu_round.sh session (gpurun_out/*_TAG*) into profiles/r01/ with
the ncu summaries (scripts/ncu_summary.py + ncu_lines.py) and the launch list
summary.  Usage: python scripts/refresh_profiles.py TAG"""
import collections, csv, json, shutil, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
g, p = ROOT / "gpurun_out", ROOT / "profiles" / "r01"
last = lambda f: (g / f).read_text().strip().splitlines()[-1] + "\n"
(p / "bench.json").write_text(last(f"bench_{tag}.json"))
(p / "bench_reference.json").write_text(last(f"bench_ref_{tag}.json"))
shutil.copy(g / f"modes_{tag}.jsonl", p / "bench_modes.jsonl")
shutil.copy(g / f"launches_{tag}.csv", p / "launches.csv")
shutil.copy(g / f"stats_{tag}.log", p / "kernel_stats.txt")
shutil.copy(g / f"e2e_{tag}.log", p / "e2e_breakdown.txt")
rows = [r for r in csv.reader(open(g / f"launches_{tag}.csv")) if len(r) > 10]
h = rows[0]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0].replace("<unnamed>::", "")[-48:]].append(float(r[vi].replace(",", "")))
with open(p / "launches_summary.txt", "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --steps 3 --warmup 3 ({tag})\n")
    for k, v in d.items():
        f.write(f"{k:50s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.1f} us\n")
def summ(rep, out, kernel=None):
    a = subprocess.run([sys.executable, str(ROOT / "scripts/ncu_summary.py"), str(rep)], capture_output=True, text=True).stdout
    b = subprocess.run([sys.executable, str(ROOT / "scripts/ncu_lines.py"), str(rep), "30"], capture_output=True, text=True).stdout
    (p / out).write_text(a + "\n# hottest source lines (all captured kernels)\n" + b)
    return a
summ(g / f"prof_march_{tag}.ncu-rep", "ncu_march_kernel.txt")
summ(g / f"prof_trace_{tag}.ncu-rep", "ncu_trace_intervals_kernel.txt")
summ(g / f"prof_march272_{tag}.ncu-rep", "ncu_march_kernel_radial272.txt")
def dram(rep):
    raw = list(csv.reader(__import__("io").StringIO(subprocess.run(
        ["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
    hh = raw[0]
    r0 = raw[2]
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    val = lambda k: float(r0[hh.index(k)].replace(",", "")) * sc.get(raw[1][hh.index(k)], 1)
    return val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
r59, w59 = dram(g / f"prof_march_{tag}.ncu-rep")
r272, w272 = dram(g / f"prof_march272_{tag}.ncu-rep")
(p / "ncu_dram.json").write_text(json.dumps({
    "kernel": "march_sm_kernel<4, 3>", "scene": "radial59 512x512 skip-adaptive",
    "dram_bytes_read": int(r59), "dram_bytes_write": int(w59), "dram_bytes_per_launch": int(r59 + w59),
    "source": f"ncu --set full, gpurun_out/prof_march_{tag}.ncu-rep (profiles/r01/ncu_march_kernel.txt; the second capture is the G=16 launch that returns at once)",
    "radial272": {"kernel": "march_sm_kernel<4, 3>", "dram_bytes_read": int(r272), "dram_bytes_write": int(w272)}},
    indent=1) + "\n")
print("ok", tag)
