"""Throughput of the q-th degree neighbourhood engine (aca_qnbr_run, P12) on
c3-shaped physics (heat-bath, beta scaled so that beta * z stays at the q = 1 critical coupling's
4 beta_c: the same acceptance regime for every q), 2-D and 3-D. A widening row: measured, not
tuned. Reported per q: arrivals/s over the device time of the sweeps (initialisation excluded),
sweeps, launches, and the bytes per cell per sweep of the engine's SoA state (13 B read + written).
usage: python scripts/qnbr_bench.py [--side 4096] [--side3 256] [--T 5] [--rounds 0]"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_cs_0502039_b200 as aca  # noqa: E402


def nbrs(ndim, q):
    return 2 * q * (q + 1) if ndim == 2 else (2 * q + 1) * (2 * q * q + 2 * q + 3) // 3 - 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=4096)
    ap.add_argument("--side3", type=int, default=256)
    ap.add_argument("--T", type=float, default=5.0)
    ap.add_argument("--rounds", type=int, default=0)
    ap.add_argument("--qs", type=str, default="1,2,3,4")
    a = ap.parse_args()
    beta_c = 0.5 * math.log(1.0 + math.sqrt(2.0))
    aca.aca_qnbr_run((64, 64), 1, 1.0, beta=beta_c, want_state=False)   # warm-up (context, module load)
    for ndim, side in ((2, a.side), (3, a.side3)):
        dims = (side,) * ndim
        n = side ** ndim
        for q in [int(v) for v in a.qs.split(",")]:
            z = nbrs(ndim, q)
            beta = beta_c * 4.0 / z
            best = None
            for rep in range(3):
                _, _, _, st = aca.aca_qnbr_run(dims, q, a.T, beta=beta, seed=1, rounds=a.rounds, want_state=False)
                if best is None or st["gpu_seconds"] < best["gpu_seconds"]:
                    best = st
            sec = best["gpu_seconds"]
            print(json.dumps({"engine": "aca_qnbr_run", "ndim": ndim, "dims": list(dims), "q": q, "members": z,
                              "T": a.T, "beta": beta, "arrivals": best["arrivals"], "flips": best["flips"],
                              "sweeps": best["sweeps"], "launches": best["launches"], "gpu_seconds": sec,
                              "arrivals_per_s": best["arrivals"] / sec,
                              "state_GBps": 26.0 * n * best["sweeps"] / sec / 1e9,
                              "event_hash": "%016x" % best["event_hash"]}), flush=True)


if __name__ == "__main__":
    main()
