"""Validate the reference arm's block sampling (bench.py --impl reference):
the reference's whole grid composition (oracle/_ref ref_grid_pipeline_timed,
best of `--reps` runs: the first run of a process pays page faults on fresh
allocations, bench_poisson also takes the best of reps) against the sum of
the 16 stock-composition blocks bench.py times as its steps, on the same
host.  Writes profiles/r2_reference_validation.json; bench.py quotes it.

ORACLE / TEST INFRASTRUCTURE: times the reference only."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_reference_validation.json"))
    args = ap.parse_args()
    import bench
    from conftest import zero_mean_noise
    from oracle.oracle import Oracle, Reference
    from paper_1510_08094_b200 import inputs
    R, O = Reference(), Oracle()
    threads = min(os.cpu_count() or 1, 16)
    res = json.load(open(args.out)) if os.path.exists(args.out) else {}
    for name in args.configs.split(","):
        cfg = inputs.CONFIGS[name]
        f = zero_mean_noise(O, cfg.M, cfg.N, 1)
        runs = []
        for _ in range(args.reps):
            _, _, tp = R.grid_pipeline_timed(f, cfg.M, threads=threads)
            runs.append(tp)
        best = min(runs, key=lambda t: t.sum())
        bsum = 0.0
        bench.reference_block(R, cfg, 0, threads)  # allocate + warm the sampler's matrices
        for b in range(bench.BLOCKS):
            s, _ = bench.reference_block(R, cfg, b, threads)
            bsum += s
        row = {"full_composition_s": float(best.sum()), "full_runs_s": [float(t.sum()) for t in runs],
               "phases_s": dict(zip(["sample_dfs", "analyze_2d", "msin2", "solve", "sample_grid"],
                                    [float(x) for x in best])),
               "blocks_sum_s": bsum, "blocks_over_full": bsum / float(best.sum()), "threads": threads,
               **bench.host_facts()}
        res[name] = row
        print(name, json.dumps(row), flush=True)
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
