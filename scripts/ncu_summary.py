"""Summarise an ncu report: key metrics, stall reasons, hottest source lines."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
def page(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(page(["--page", "raw", "--csv"]))))
h, u = raw[0], raw[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum", "lts__t_bytes.sum"]
for row in raw[2:]:
    print("----")
    for k in want:
        if k in h:
            i = h.index(k)
            print(f"  {k} = {row[i]} {u[i]}")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(row[i]), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(s for s, _ in st) or 1
    print("  stalls:", ", ".join(f"{n} {100*s/tot:.1f}%" for s, n in sorted(st, reverse=True)[:8]))
if len(sys.argv) > 2:
    src = list(csv.reader(io.StringIO(page(["--page", "source", "--csv", "--print-source=cuda,sass"]))))
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ""])
    for r in src[3:]:
        if len(r) < 9 or r[0] == "Line No" or r[2] != "-":
            continue
        try:
            a = agg[int(r[0])]
            a[0] += float(r[4] or 0); a[1] += float(r[7] or 0); a[2] += float(r[8] or 0); a[3] = r[1][:90]
        except ValueError:
            pass
    tot = sum(v[0] for v in agg.values()) or 1
    for ln, v in sorted(agg.items(), key=lambda x: -x[1][0])[: int(sys.argv[2])]:
        eff = v[2] / v[1] if v[1] else 0
        print(f"{100*v[0]/tot:5.1f}% L{ln:4d} thr/inst={eff:5.1f} inst={v[1]:11.0f}  {v[3]}")
