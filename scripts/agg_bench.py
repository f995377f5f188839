"""Throughput of the aggregated Poisson-stream engine (fig:amcpoi) on BASELINE config-3-shaped
input (16384^2 heat-bath at beta_c, T = 20) for several subarray sizes m, next to the main
per-cell path. usage: python scripts/agg_bench.py [--T 20] [--budget 64]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_cs_0502039_b200 as aca  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=float, default=20.0)
    ap.add_argument("--dims", type=str, default="16384x16384")
    ap.add_argument("--budget", type=int, default=64)
    a = ap.parse_args()
    dims = tuple(int(v) for v in a.dims.split("x"))
    for m in (8, 4, 2):
        aca.aca_agg_run((256, 256), m, 1.0, beta=0.4406868, want_state=False)   # warm-up
        _, _, _, st = aca.aca_agg_run(dims, m, a.T, beta=0.4406868, seed=1, budget=a.budget, want_state=False)
        print(json.dumps({"algorithm": "fig:amcpoi aggregated stream", "m": m, "dims": list(dims), "T": a.T,
                          "arrivals": st["arrivals"], "launches": st["launches"], "gpu_seconds": st["gpu_seconds"],
                          "arrivals_per_s": st["arrivals"] / st["gpu_seconds"]}), flush=True)


if __name__ == "__main__":
    main()
