"""Summarise an ncu source page (`--page source --csv --print-source cuda,sass`)
per CUDA source line: stall samples and warp instructions executed."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur = None; hdr = None; agg = {}
def f(x):
    try: return float(x)
    except: return 0.0
for r in rows:
    if not r: continue
    if r[0] in ("File Path", "File Name"): cur = r[1].split('/')[-1]; continue
    if r[0] in ("Function Name", "Kernel Name"): continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or not r[0].strip().isdigit(): continue
    i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_i = hdr.index("Instructions Executed")
    a = agg.setdefault((cur, int(r[0])), [0, 0, r[1][:90]])
    a[0] += f(r[i_s]); a[1] += f(r[i_i])
tot = sum(v[0] for v in agg.values()) or 1; toti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot:.0f}, warp instructions {toti:.3e}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 0
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:n]:
    print(f"{k[0]}:{k[1]:4d} samp {100*v[0]/tot:5.1f}% inst {100*v[1]/toti:5.1f}%  {v[2]}")
