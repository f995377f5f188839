"""Reproduce the paper's time-only efficiency experiment (fig:perf1t1) on
the GPU at sizes far beyond the paper's: for each topology (n-circle, n x n torus, n^3 cube)
and asynchrony law (Poisson, uniform, r^(1/8)), S independent runs (different seeds), the
steady-state mean of N0/N per run, and a 99.99% Student confidence interval over the runs (the
paper's method). Also the achieved HBM bandwidth of the iteration kernel
(algorithmic bytes: one 8-byte read and one 8-byte write of t per cell and iteration).
usage: python scripts/efficiency.py [--runs S] [--rounds R] [--warmup W] [--out file.json]"""
import argparse
import json
import os
import sys

import numpy as np
from scipy import stats

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_cs_0502039_b200 as aca  # noqa: E402

PAPER = {(1, 0): "0.247", (1, 1): "0.271", (1, 2): "0.3388 +- 0.0012", (2, 0): "about 0.121", (2, 1): "about 0.132"}
LAWS = ["Poisson", "uniform", "r^(1/8)"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=600)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    shapes = {1: (1 << 28,), 2: (16384, 16384), 3: (512, 512, 512)}
    rows = []
    for nd in (1, 2, 3):
        for law in (0, 1, 2):
            dims = shapes[nd]
            n = int(np.prod(dims))
            means, secs = [], []
            for s in range(a.runs):
                fired, sec = aca.aca_efficiency_run(dims, a.rounds, law=law, seed=1000 * nd + 100 * law + s)
                means.append(float((fired[a.warmup:].astype(np.float64) / n).mean()))
                secs.append(sec)
            m = float(np.mean(means))
            hw = float(stats.t.ppf(1 - 0.0001 / 2, a.runs - 1) * np.std(means, ddof=1) / np.sqrt(a.runs)) if a.runs > 1 else None
            gbs = n * 16 * a.rounds / float(np.mean(secs)) / 1e9
            row = {"ndim": nd, "dims": list(dims), "law": LAWS[law], "efficiency": m, "ci99.99_halfwidth": hw,
                   "runs": a.runs, "rounds": a.rounds, "warmup": a.warmup, "paper": PAPER.get((nd, law)),
                   "iteration_ms": 1e3 * float(np.mean(secs)) / a.rounds,
                   "cell_iterations_per_s": n * a.rounds / float(np.mean(secs)),
                   "hbm_gbs_algorithmic": gbs, "hbm_frac": gbs / peak}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.out:
        json.dump({"rows": rows, "peak_gbs": peak}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
