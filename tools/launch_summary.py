"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`)
into per-kernel counts, mean durations and shares (markdown)."""
import collections, csv, sys


def main(path, out):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr, data = None, []
    for r in rows:
        if r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
        agg.setdefault(name, []).append(float(d["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list: `{path.split('/')[-1]}`", "",
             f"{len(data)} launches, {tot / 1e3:.3f} ms total (cold-cache, serialised replay; shares are what count)", "",
             "| kernel | launches | mean µs | total ms | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v) / 1e3:.3f} | {100 * sum(v) / tot:.1f}% |")
    step = [k for k in agg if any(s in k for s in ("lambda_fwd", "theta", "lambda_inv"))]
    if step:
        per = {k: sum(agg[k]) / len(agg[k]) for k in step}
        st = sum(per.values())
        lines += ["", "Share of one solve step (mean launch time of each solver kernel; input generation",
                  "and the torch parity checks are outside the timed region):", "",
                  "| kernel | mean µs | step share |", "|---|---|---|"]
        lines += [f"| {k} | {v:.1f} | {100 * v / st:.1f}% |" for k, v in per.items()]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
