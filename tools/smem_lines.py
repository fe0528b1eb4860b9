"""Per-CUDA-line shared-memory wavefronts (actual vs ideal) of one kernel from an ncu
report (developer tool): python tools/smem_lines.py rep.ncu-rep kernel_regex [top]"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
agg = collections.OrderedDict(); src = {}
h = None; fn = None
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "File Path": fn = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        h = r; iw = h.index("L1 Wavefronts Shared"); ii = h.index("L1 Wavefronts Shared Ideal")
        ig = h.index("L1 Tag Requests Global"); continue
    if h is None or len(r) <= iw or not r[0].strip().isdigit(): continue
    key = (fn, int(r[0])); src[key] = r[1].strip()[:80]
    try: w = float(r[iw] or 0); i = float(r[ii] or 0); g = float(r[ig] or 0)
    except ValueError: continue
    a = agg.setdefault(key, [0, 0, 0]); a[0] += w; a[1] += i; a[2] += g
tw = sum(v[0] for v in agg.values()) or 1
print(f"shared wavefronts {tw:.4g} (ideal {sum(v[1] for v in agg.values()):.4g}), global tag requests {sum(v[2] for v in agg.values()):.4g}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:<5d} {100 * v[0] / tw:5.1f}% wf {v[0]:.3g} ideal {v[1]:.3g} | {src.get(k, '')}")
