"""Throughput of the aggregated engines — fig:amcpoi (one Poisson stream per subarray) and the
modified BKL — on BASELINE-shaped inputs, next to the per-cell path.
Reported: events/s (stream arrivals; BKL skips kernel rejections, so it has fewer events) and
the attempt-equivalent rate N lambda T / seconds (simulated cell-time per second), the number
that compares algorithms with different event definitions.
usage: python scripts/agg_bench.py [--config c3|c5] [--budget 64]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_cs_0502039_b200 as aca  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--budget", type=int, default=64)
    ap.add_argument("--ms", type=str, default="8,4")
    a = ap.parse_args()
    cfg = workloads.config(a.config)
    dims, T = tuple(cfg["dims"]), cfg["T"]
    n = dims[0] * dims[1]
    kw = dict(lam=cfg["lam"], beta=cfg["beta"], J=cfg["J"], h=cfg["h"], rule=cfg["rule"], init_q=cfg["init_q"])
    for bkl in (False, True):
        for m in [int(v) for v in a.ms.split(",")]:
            aca.aca_agg_run((256, 256), m, 1.0, want_state=False, bkl=bkl, **kw)   # warm-up
            _, _, _, st = aca.aca_agg_run(dims, m, T, seed=1, budget=a.budget, want_state=False, bkl=bkl, **kw)
            sec = st["gpu_seconds"]
            print(json.dumps({"config": a.config, "algorithm": "modified BKL" if bkl else "fig:amcpoi stream",
                              "m": m, "dims": list(dims), "T": T, "events": st["arrivals"], "flips": st["flips"],
                              "launches": st["launches"], "gpu_seconds": sec, "events_per_s": st["arrivals"] / sec,
                              "attempt_equivalent_per_s": n * cfg["lam"] * T / sec}), flush=True)


if __name__ == "__main__":
    main()
