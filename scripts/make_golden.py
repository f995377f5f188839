"""Write tests/golden/<config>_seed<k>.json: SHA-256 digests of the final spins, times and
counters plus the integer statistics of a FULL oracle run of a BASELINE config.
Calls only oracle/ (the serial PQ oracle); nothing here touches the CUDA path.
usage: python scripts/make_golden.py c2 [seed] [T'[,T''...]] [--calendar]
With T' (< the config's T; "-" = the config's T) the run stops at T' and the file is
<config>_seed<k>_T<T'>.json: an interim full-lattice digest for configs whose full-T oracle run
takes hours. A comma-separated list of horizons writes one file per horizon from ONE run
(run_until composes); the config's own T in the list writes the full file. --calendar runs the oracle's calendar-queue form of the same priority queue (the same
event order, pinned equal to the binary heap by tests/test_oracle_sim.py; faster on big lattices)."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def write(name, seed, cfg, T, o, t0, calendar):
    st = o.stats()
    st.pop("rounds")
    interim = T != cfg["T"]
    out = {"config": name, "seed": seed, "dims": list(cfg["dims"]), "T": T,
           "generated_by": "scripts/make_golden.py (oracle/ only)",
           "queue": "calendar (D)" if calendar else "binary heap (A)", "oracle_seconds": round(time.time() - t0, 1),
           "sha256_spins_int8": digest(o.spins()), "sha256_times_u64": digest(o.times()),
           "sha256_counters_u32": digest(o.counters()), "stats": {k: int(v) for k, v in st.items()}}
    stem = "%s_seed%d" % (name, seed) + ("_T%g" % T if interim else "")
    path = os.path.join(ROOT, "tests", "golden", stem + ".json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, out["oracle_seconds"], "s", flush=True)


def main():
    calendar = "--calendar" in sys.argv
    argv = [a for a in sys.argv if a != "--calendar"]
    name = argv[1]
    seed = int(argv[2]) if len(argv) > 2 else workloads.PARITY_SEEDS[0]
    cfg = workloads.config(name)
    horizons = [cfg["T"]]
    if len(argv) > 3 and argv[3] != "-":
        horizons = sorted(float(x) for x in argv[3].split(","))
    assert all(T <= cfg["T"] for T in horizons), "a horizon beyond the config's T"
    t0 = time.time()
    o = oracle.OracleSim(cfg["dims"], lam=cfg["lam"], beta=cfg["beta"], J=cfg["J"], h=cfg["h"], rule=cfg["rule"],
                         seed=seed, init_q=cfg["init_q"])
    for T in horizons:
        o.run_until(T, order="calendar" if calendar else "pq")
        write(name, seed, cfg, T, o, t0, calendar)


if __name__ == "__main__":
    main()
