"""Launch list (ncu --metrics gpu__time_duration.sum --csv) -> per-launch ms in order
and per-kernel totals (developer tool): python tools/launch_list.py file.csv [min_ms]"""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(r for r in rows if "Kernel Name" in r)
kn, mv, mn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
lo = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
seq = []
for r in rows[rows.index(h) + 1:]:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum": continue
    t = float(r[mv].replace(",", "")) / 1e6  # ns -> ms
    seq.append((r[kn].split("(")[0].replace("void ", "").replace("nmx::", ""), t))
tot = sum(t for _, t in seq)
print(f"{len(seq)} launches, {tot:.3f} ms")
for n, t in seq:
    if t >= lo: print(f"{t:8.3f}  {n[:100]}")
agg = collections.Counter()
for n, t in seq: agg[n.split("<")[0]] += t
print("per kernel:")
for n, t in agg.most_common(): print(f"{t:8.3f}  {n}")
