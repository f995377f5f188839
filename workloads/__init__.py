"""Seeded synthetic workloads shared by the tests, bench.py and the oracle legs.

Holds only parameters and seeded input arrays — none of the method's arithmetic (no
Philox, no -ln, no flip table, no firing rule). Both the CUDA path and the oracle receive
what is built here. The five configurations are BASELINE.json `configs` (the paper uses
synthetic tori only: 120^2, 128^2, 384^2; these scale them).
"""
import numpy as np

HEATBATH, METROPOLIS = 0, 1

CONFIGS = {
    "c1": dict(dims=(64, 64), beta=0.4406868, J=1.0, h=0.0, lam=1.0, rule=HEATBATH,
               init_q=0.5, T=10.0, tile=(64, 64), note="one cell per PE rule; whole lattice = one CTA"),
    "c2": dict(dims=(1024, 1024), beta=0.40, J=1.0, h=0.0, lam=1.0, rule=METROPOLIS,
               init_q=0.5, T=100.0, tile=(64, 64), note="single B200, 64x64 CTA tiles, 1-cell halo (resident in shared memory across sweeps)",
               opts={"rounds_per_launch": 6}),   # 256 tiles only: more rounds per visit (measured best)
    "c3": dict(dims=(16384, 16384), beta=0.4406868, J=1.0, h=0.0, lam=1.0, rule=HEATBATH,
               init_q=0.5, T=20.0, tile=(64, 64), note="row strips across 1/2/4/8 GPUs"),
    "c4": dict(dims=(512, 512, 512), beta=0.2216544, J=1.0, h=0.0, lam=1.0, rule=HEATBATH,
               init_q=0.5, T=10.0, tile=(32, 16, 8), note="z slabs across 1/2/4/8 GPUs"),
    "c5": dict(dims=(8192, 8192), beta=1.0, J=1.0, h=0.1, lam=1.0, rule=METROPOLIS,
               init_q=0.05, T=200.0, tile=(64, 64),
               note="low temperature; exact early rejection, path chosen per tile from its BKL class histogram",
               opts={"early_reject": 1, "class_book": 1, "class_wmax": 0.01}),
}

PARITY_SEEDS = (1, 2, 3)
TIMING_SEED = 1


def config(name, **override):
    c = dict(CONFIGS[name])
    c.update(override)
    return c


def scaled(name, dims, T=None):
    """The same physics (beta, h, rule, init) on a smaller lattice / shorter horizon."""
    c = config(name)
    c["dims"] = tuple(dims)
    if T is not None:
        c["T"] = float(T)
    return c


def host_spins(dims, seed, q_minus=0.5):
    """A seeded i.i.d. +-1 configuration (numpy PCG64, unrelated to the method's Philox
    streams) used as a user-supplied initial state, e.g. for the end-to-end bench leg."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = int(np.prod(dims))
    return np.where(rng.random(n) < q_minus, -1, 1).astype(np.int8)
