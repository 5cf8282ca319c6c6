"""Summarise ncu reports into profiles/: per-kernel key metrics, DRAM traffic
per launch, top stall reasons and hottest source lines (markdown + JSON)."""
import csv, io, json, subprocess, sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["__units"] = dict(zip(hdr, units))
        kernels.append(d)
    return hdr, kernels


SCALE = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1.0}


KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main(rep, out_prefix):
    hdr, ks = raw_metrics(rep)
    summary = []
    for d in ks:
        e = {"kernel": d.get("Kernel Name", "")[:60]}
        for k, name in KEYS.items():
            if k in d:
                v = num(d[k])
                u = d["__units"].get(k, "")
                if v is not None and u in SCALE:
                    v *= SCALE[u]
                e[name] = v
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v) for h, v in d.items()
                  if isinstance(v, str) and h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        tot = sum(v for v in stalls.values() if v) or 1
        e["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0))[:6] if v}
        if e.get("dram_read_bytes") is not None:
            e["dram_bytes"] = (e.get("dram_read_bytes") or 0) + (e.get("dram_write_bytes") or 0)
            if e.get("duration_ns"):
                e["dram_gbs"] = e["dram_bytes"] / e["duration_ns"]
        summary.append(e)
    with open(out_prefix + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    with open(out_prefix + ".md", "w") as fh:
        fh.write(f"# ncu summary of `{rep.split('/')[-1]}`\n\n")
        for e in summary:
            fh.write(f"## {e['kernel']}\n\n")
            for k, v in e.items():
                if k != "kernel":
                    fh.write(f"- {k}: {v}\n")
            fh.write("\n")
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
