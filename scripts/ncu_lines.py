"""Per-source-line instruction counts and stall samples of an ncu report
(ncu -i REP --page source --print-source cuda,sass)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 45
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, out = None, []
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        try:
            out.append((int(r[7]), int(r[4]), fn, int(r[0]), r[1][:90]))
        except ValueError:
            pass
ti = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
print(f"total warp-instructions {ti / 1e6:.1f}M, stall samples {ts}")
files = {}
for i, s, f, _, _ in out:
    a = files.setdefault(f, [0, 0]); a[0] += i; a[1] += s
for f, (i, s) in sorted(files.items(), key=lambda x: -x[1][0]):
    print(f"  {f}: {100 * i / ti:.1f}% inst, {100 * s / ts:.1f}% stalls")
for i, s, f, l, src in sorted(out, reverse=True)[:top]:
    print(f"{i / 1e6:7.2f}M {100 * i / ti:5.1f}%i {100 * s / ts:5.1f}%s {f}:{l} {src}")
