"""Summarise an ncu source page (cuda,sass CSV) per CUDA source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur = None; hdr = None; agg = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] in ("Function Name", "Kernel Name"): continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or not r[0].strip().isdigit(): continue
    d = dict(zip(hdr, r))
    def f(x):
        try: return float(x)
        except: return 0.0
    a = agg.setdefault((cur, int(r[0])), [0, 0, r[1][:100]])
    a[0] += f(r[4]); a[1] += f(r[7])
tot = sum(v[0] for v in agg.values()) or 1; toti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot:.0f}, warp instructions {toti:.3e}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k[0]}:{k[1]:4d} samp {100*v[0]/tot:5.1f}% inst {100*v[1]/toti:5.1f}%  {v[2]}")
