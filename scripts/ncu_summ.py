"""Summarise an ncu raw/details/sass CSV triple (as written by scripts/gpu_r2v.sh)."""
import csv, gzip, io, sys
from collections import Counter

n = sys.argv[1]
rows = list(csv.reader(open(f"{n}_raw.csv")))
v = dict(zip(rows[0], rows[2])); u = dict(zip(rows[0], rows[1]))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    for h in v:
        if h == k or (h.startswith(k) and h.count('.') == k.count('.')):
            print("  ", h, u[h], v[h])
items = [(h, float(v[h])) for h in v if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
print("  stalls:", ", ".join("%s %.2f" % (h.split("stalled_")[1].split("_per")[0], x) for h, x in sorted(items, key=lambda t: -t[1])[:8]))
try:
    rows = list(csv.reader(io.TextIOWrapper(gzip.open(f"{n}_sass.csv.gz"))))
except FileNotFoundError:
    sys.exit()
h = rows[1]; data = rows[2:]
iS = h.index("Source"); iW = h.index("Warp Stall Sampling (All Samples)"); iE = h.index("Instructions Executed")
c = Counter(); ni = Counter()
for r in data:
    e = int(r[iE] or 0); w = int(r[iW] or 0)
    c[e] += w; ni[e] += e
tot = sum(c.values())
print("  samples by exec-count bucket (count: samples%, instructions):")
for e, w in c.most_common(10):
    print("    %9d: %5.1f%% %d" % (e, 100.0 * w / tot, ni[e]))
