import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = {}
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.setdefault(d['ID'] + ' ' + d['Kernel Name'][:22], {})[d['Metric Name']] = d['Metric Value']
for k, v in out.items():
    t = float(v['gpu__time_duration.sum']) / 1e6
    rb = float(v['dram__bytes_read.sum']) / 1e9; wb = float(v['dram__bytes_write.sum']) / 1e9
    print(f"{k:28s} {t:7.2f} ms  R {rb:6.2f} GB W {wb:6.2f} GB  {(rb + wb) / (t * 1e-3):6.0f} GB/s  warps {float(v['sm__warps_active.avg.pct_of_peak_sustained_active']):5.1f}%  occ-lim reg {v.get('launch__occupancy_limit_registers')} smem {v.get('launch__occupancy_limit_shared_mem')}")
