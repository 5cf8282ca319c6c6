"""cuFFT comparison point (torch.fft, FP64) on the shapes of the grid path.

The north star times cuFFT only as a comparison for the hand-written
transforms.  For each config this measures, with CUDA events after warm-up:

  rfft_rows   torch.fft.rfft over the (M/2+1) x N real physical rows
              (cuFFT D2Z; our lambda_fwd also does the DFS sign, the 1/N and
              the transpose to mode-major order)
  fft_cols    torch.fft.fft + ifft over (N/2+1) doubled columns of length M
              (cuFFT Z2Z, forward + inverse: the transform work of our theta
              stage, which also folds the DFS symmetry, applies Msin^2 and runs
              the banded solves between the two transforms)
  irfft_rows  torch.fft.irfft back to the real rows (cuFFT Z2D)

and prints one JSON line per config with our own per-stage times from the
same run (Plan.stage_times, CUDA events on the plan stream).

    python tools/cufft_compare.py [C2 C3 C4] > profiles/r1_cufft_compare.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1510_08094_b200 import inputs  # noqa: E402
from paper_1510_08094_b200.poisson import Plan  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), statistics.median(ts)


def main(names):
    dev = torch.device("cuda")
    for name in names:
        cfg = inputs.CONFIGS[name]
        M, N, nr = cfg.M, cfg.N, cfg.nrhs
        R, C = M // 2 + 1, N // 2 + 1
        g = torch.Generator(device="cuda").manual_seed(1)
        rows = torch.randn((nr, R, N), generator=g, device=dev, dtype=torch.float64)
        res = {"config": name, "M": M, "N": N, "nrhs": nr}
        spec = torch.fft.rfft(rows, dim=-1)
        res["cufft_rfft_rows_ms"] = timed(lambda: torch.fft.rfft(rows, dim=-1))[0]
        res["cufft_irfft_rows_ms"] = timed(lambda: torch.fft.irfft(spec, n=N, dim=-1))[0]
        del spec
        cols = torch.complex(torch.randn((nr, C, M), generator=g, device=dev, dtype=torch.float64),
                             torch.randn((nr, C, M), generator=g, device=dev, dtype=torch.float64))
        res["cufft_fft_ifft_cols_ms"] = timed(lambda: torch.fft.ifft(torch.fft.fft(cols, dim=-1), dim=-1))[0]
        del cols
        res["cufft_transforms_ms"] = res["cufft_rfft_rows_ms"] + res["cufft_fft_ifft_cols_ms"] + res["cufft_irfft_rows_ms"]
        # our solve on the same config (device-resident, stage times from CUDA events)
        with Plan(M, N, nr) as plan:
            f = torch.empty((nr, R, N) if nr > 1 else (R, N), dtype=torch.float64, device=dev)
            c = torch.from_numpy(inputs.sh_coeffs(1, cfg.L, cfg.p)).to(dev)
            if nr > 1:
                for r in range(nr):
                    plan.shgen(cfg.L, c, f[r])
            else:
                plan.shgen(cfg.L, c, f)
            u = torch.empty_like(f)
            plan.set_stream(torch.cuda.current_stream().cuda_stream)
            res["ours_solve_ms"] = timed(lambda: plan.solve_grid(f, u))[0]
            plan.enable_stage_timing(True)
            acc = {}
            for _ in range(5):
                plan.solve_grid(f, u)
                for k, v in plan.stage_times().items():
                    acc[k] = acc.get(k, 0.0) + v / 5
            plan.enable_stage_timing(False)
            res["ours_stage_ms"] = acc
        res["note"] = ("cuFFT columns are the doubled length-M columns without the DFS doubling copy, the "
                       "transposes or the solve; ours includes all of them")
        print(json.dumps(res), flush=True)
        del rows, f, u
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3", "C4"])
