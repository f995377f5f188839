#!/usr/bin/env python
"""Benchmark of the conservative Poisson-asynchronous Ising path (BASELINE.json metric:
Poisson arrivals processed/s at 1/2/4/8 B200; achieved HBM GB/s vs peak).

One step = the whole hot path on one batch of synthetic input: P5 initialisation on the
device (aca_reset), aca_run_until(T) (all in-tile rounds / outer rounds / halo exchanges),
aca_get_stats (device reductions of B, M, arrivals). Default workload: config 3 (2-D
16384^2 heat-bath at beta_c, T = 20, row strips across the GPUs) — the configuration the
metric's 1->8 GPU scaling and HBM target are quoted on. State (3.2 GB) >> L2 (126 MB).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]
Under torchrun (N > 1) each rank owns a row strip; time = max over ranks; rank 0 prints.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

METRIC = "Poisson arrivals processed/sec"
UNIT = "arrivals/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--seed", type=int, default=workloads.TIMING_SEED)
    ap.add_argument("--rounds", type=int, default=0, help="in-tile rounds per launch (0 = library default)")
    ap.add_argument("--tile", type=str, default="", help="e.g. 64x64 or 32x16x8")
    ap.add_argument("--launches-per-check", type=int, default=0)
    ap.add_argument("--early-reject", type=int, default=-1, help="a10 early rejection (-1 = config default)")
    ap.add_argument("--class-book", type=int, default=-1, help="a10 per-tile class bookkeeping (-1 = config default)")
    ap.add_argument("--class-wmax", type=float, default=None, help="a10 path iff a tile's mean flip probability <= this")
    ap.add_argument("--checkerboard", type=int, default=0, help="1/0 = checkerboard sweeps (default), -1 = off")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="N>1 halo transport: kernel stores into CUDA-IPC-mapped neighbour halos (push "
                         "mode, default) or NCCL send/recv between launches")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-hash", action="store_true", help="skip the P7 event hash (diagnostics only)")
    ap.add_argument("--rows-div", type=int, default=1,
                    help="run the config on 1/G of its rows (2-D) / planes (3-D): the per-GPU lattice of a G-GPU "
                         "strip partition, to bound the per-GPU launch/tail cost of the multi-GPU runs on one device")
    ap.add_argument("--shards", type=int, default=1,
                    help="virtual row strips / z slabs on this GPU (bounds the per-shard boundary cost of the "
                         "multi-GPU partition on one device; push-mode halos, same kernels)")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks during the timed region
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy b.copy_(a))"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_entry(config):
    """The committed ncu --set full summary of this config's tile kernel
    (profiles/ncu_full_summary.json, keyed by config; written by scripts/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        return json.load(open(p)).get(config)
    except Exception:
        return None


def ncu_traffic(config):
    """dram bytes per launch of the tile kernel from this config's committed ncu capture."""
    d = ncu_entry(config) or {}
    return d.get("dram_bytes_per_launch")


def l2_copy_gbs(torch):
    """Measured L2 bandwidth for the L2-resident config: torch copy_ between two 16 MiB buffers
    (both stay in the 126 MB L2), read + write bytes, best of 20 (CUDA events)."""
    a = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    best = 0.0
    for _ in range(3):
        b.copy_(a)
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 50 * 2 * a.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def issue_roofline(config):
    """Secondary roofline of the tile kernel, which is issue/ALU-bound: warp instructions issued
    per second in the committed ncu --set full capture against the issue limit of the chip
    (4 SMSPs x 1 warp-instruction/cycle per SM, B300_MICROARCH.md 'Per-warp issue scheduler';
    148 SMs at the captured SM clock)."""
    try:
        d = ncu_entry(config) or {}
        inst, ms, clk = d["warp_inst_per_launch"], d["launch_ms"], d["sm_clock_hz"]
        ach = inst / (ms * 1e-3)
        peak = 148 * 4 * clk
        return {"bound": "issue", "achieved": ach, "peak": peak, "unit": "warp-inst/s", "frac": ach / peak,
                "alu_pipe_frac": d.get("alu_pipe_pct", 0) / 100.0, "source": d.get("source"),
                "note": "measured under ncu (cold cache, serialised), not in this run"}
    except Exception:
        return None


def algorithmic_bytes_per_cell(ndim, tile):
    """Per sweep (in place, 1-cell halo): read each cell's packed word (t, n, s: 8 B) and write it
    back (8 B), plus the halo words of the tile faces. DESIGN.md 'Roofline' (the builder's
    convention; SURVEY.md section 8(d) counts 13 B/cell SoA state instead: SURVEY_BYTES)."""
    if ndim == 2:
        tx, ty = tile[0], tile[1]
        halo = 8.0 * 2 * (tx + ty) / (tx * ty)
    else:
        tx, ty, tz = tile
        halo = 8.0 * 2 * (tx * ty + ty * tz + tx * tz) / (tx * ty * tz)
    return 16.0 + halo


# bytes per cell per outer round of the SoA layout it assumed (t, n, s:
# 13 B read + 13 B written, + 0.56 B tile-halo re-read for 64^2 tiles; 3-D tiles 29.4 B)
SURVEY_BYTES = {2: 26.6, 3: 29.4}


def oracle_sample(cfg, seconds_target=10.0):
    """The oracle as it stands on a bounded sample of the workload: the same physics (beta, h,
    rule, init) on a lattice larger than the host's caches (2-D 4096 x 2048, 3-D 256 x 256 x 128,
    or the whole lattice if smaller), run to T' = min(T, the time that gives ~2.5e6 arrivals per
    second of target), on ONE core (the process is pinned to one CPU for the call).
    Returns (arrivals/s, arrivals, seconds, sample text)."""
    import oracle
    dims = tuple(cfg["dims"])
    big = seconds_target >= 8
    if len(dims) == 2:
        sdims = (min(dims[0], 4096 if big else 2048), min(dims[1], 2048 if big else 1024))
    else:
        sdims = (min(dims[0], 256), min(dims[1], 256 if big else 128), min(dims[2], 128 if big else 64))
    n = 1
    for d in sdims:
        n *= d
    T = min(cfg["T"], max(0.5, round(2.5e6 * seconds_target / (n * cfg["lam"]), 2)))
    o = oracle.OracleSim(sdims, lam=cfg["lam"], beta=cfg["beta"], J=cfg["J"], h=cfg["h"], rule=cfg["rule"],
                         seed=1, init_q=cfg["init_q"])
    old = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    core = min(old) if old else None
    if old:
        os.sched_setaffinity(0, {core})
    try:
        t0 = time.perf_counter()
        o.run_until(T)
        dt = time.perf_counter() - t0
    finally:
        if old:
            os.sched_setaffinity(0, old)
    arr = o.stats()["arrivals"]
    o.close()
    return arr / dt, arr, dt, ("oracle (serial binary-heap PQ, 1 thread pinned to CPU %s) on a %s lattice (%.0f MB of "
                               "state), same beta/h/rule/init, T'=%g of T=%g: %d arrivals in %.2f s" % (
                                   core, "x".join(map(str, sdims)), n * 13 / 1e6, T, cfg["T"], arr, dt))


def cpu_name():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, rank, world):
    """--impl reference: the oracle (serial CPU) as the reference arm, rank 0 only."""
    if rank != 0:
        return
    cfg = workloads.config(args.config)
    for _ in range(args.warmup):
        oracle_sample(cfg, 2.0)
    tot_arr, tot_t, sample = 0, 0.0, ""
    for _ in range(args.steps):
        _, arr, dt, sample = oracle_sample(cfg, 2.0)
        tot_arr += arr
        tot_t += dt
    v = tot_arr / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "config": {"workload": args.config + ": " + cfg["note"], "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu": cpu_name(), "host_cores": os.cpu_count()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_cs_0502039_b200 as aca
    from paper_cs_0502039_b200 import dist as adist

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    # ACA_BENCH_SHARED_GPU=1 (plumbing check only): every rank on cuda:0 with a gloo process
    # group, so the N > 1 path (partition, IPC push transport, reductions) runs on one GPU.
    # Its numbers are time-sliced and meaningless; the driver never sets it.
    shared = os.environ.get("ACA_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as tdist
        if shared:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workloads.config(args.config)
    dims = tuple(cfg["dims"])
    if args.rows_div > 1:
        dims = dims[:-1] + (dims[-1] // args.rows_div,)
    ndim = len(dims)
    tile = tuple(int(x) for x in args.tile.split("x")) if args.tile else tuple(cfg["tile"])
    opts = dict(init_q=cfg["init_q"], device=local, tile=tile, event_hash=0 if args.no_hash else 1)
    if args.shards > 1:
        if world > 1:
            raise SystemExit("--shards is a single-process mode (virtual shards on one GPU)")
        opts["shards"] = args.shards
    opts.update(cfg.get("opts", {}))
    if args.early_reject >= 0:
        opts["early_reject"] = args.early_reject
    if args.class_book >= 0:
        opts["class_book"] = args.class_book
    if args.class_wmax is not None:
        opts["class_wmax"] = args.class_wmax
    if args.rounds:
        opts["rounds_per_launch"] = args.rounds
    if args.launches_per_check:
        opts["launches_per_check"] = args.launches_per_check
    if args.checkerboard:
        opts["checkerboard"] = args.checkerboard
    stream = torch.cuda.Stream()            # non-default stream: the library captures CUDA graphs on it
    torch.cuda.set_stream(stream)
    opts["stream"] = stream.cuda_stream
    if world > 1:
        adist.partition(dims, world)
        opts.update(world=world, rank=rank)
        if args.transport == "nccl":
            uid = aca.aca_nccl_unique_id() if rank == 0 else bytes(128)
            opts.update(nccl_id=adist.broadcast_bytes(uid), halo_mode=1)
    sim = aca.Sim(dims, lam=cfg["lam"], beta=cfg["beta"], J=cfg["J"], h=cfg["h"], rule=cfg["rule"],
                  seed=args.seed, **opts)
    if world > 1 and args.transport == "ipc":
        failed = 0
        try:
            adist.ipc_connect(sim.handle)
        except aca.AcaError as e:   # e.g. no peer mapping between these GPUs
            failed = 1
            print("rank %d: CUDA-IPC push transport unavailable (%s)" % (rank, e), file=sys.stderr)
        if adist.reduce_sum_int(failed) > 0:
            # no silent switch of transport: the NCCL exchange is a different (slower) schedule,
            # so a number measured with it must be asked for explicitly (--transport nccl)
            raise SystemExit("CUDA-IPC push transport unavailable on some rank; rerun with --transport nccl")
    n_local = aca.aca_num_cells(sim.handle)

    def step(seed):
        sim.reset(seed)
        sim.run_until(cfg["T"])
        return sim.stats()

    for w in range(args.warmup):
        step(args.seed + 1000 + w)
    torch.cuda.synchronize()
    st0 = sim.stats()
    clocks = ClockSampler(local)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    arrivals = tested = fired = launches = kl = 0
    v_early = v_plain = 0
    ks = 0.0
    for k in range(args.steps):
        st = step(args.seed + k)
        v_early += st["tile_visits_early"]
        v_plain += st["tile_visits_plain"]
        arrivals += st["arrivals"]
        tested += st["cells_tested"]
        fired += st["cells_fired"]
        launches += st["launches"] // max(1, args.shards)   # every virtual shard counts its own sweeps
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    st1 = sim.stats()
    elapsed = e0.elapsed_time(e1) * 1e-3
    ks = st1["kernel_seconds"] - st0["kernel_seconds"]
    kl = st1["kernel_launches"] - st0["kernel_launches"]
    if world > 1:
        elapsed = adist.reduce_max(elapsed)
        arrivals = adist.reduce_sum_int(arrivals)
    value = arrivals / elapsed

    # roofline of the dominant kernel (the tile kernel): algorithmic bytes / mean time. `launches`
    # (ctl) counts outer rounds = sweeps; with checkerboard sweeps a sweep is two kernel
    # launches over half the tiles each, so bytes/sweep over sweep time = bytes/launch over
    # launch time.
    peak, peak_src = peaks()
    bpc = algorithmic_bytes_per_cell(ndim, tile)
    mean_sweep = ks / max(1, launches)
    kl_per_sweep = (kl / max(1, launches * 1.0)) if launches else 1.0
    achieved = (n_local * bpc / mean_sweep) / 1e9 if mean_sweep > 0 else None
    resident = kl_per_sweep < 0.5     # one cooperative launch per run_until: the resident-tile kernel
    tag = "res_kernel (2-D, tiles resident in shared memory, one cooperative launch per run_until)" if resident \
        else "tile_grp_kernel (%d-D)" % ndim
    traffic = ncu_traffic(args.config)
    state_bytes = n_local * 8
    l2_resident = state_bytes * 2 < 64e6          # config 2: 8 MB of state, far below the 126 MB L2
    if l2_resident:
        peak, peak_src = l2_copy_gbs(torch), "measured in this run: L2-resident torch copy_ (2 x 16 MiB)"
    sbytes = SURVEY_BYTES[ndim]
    achieved_s = (n_local * sbytes / mean_sweep) / 1e9 if mean_sweep > 0 else None
    # primary: SURVEY.md 8(d)'s per-unit figure (the contract's algorithmic bytes); beside it the
    # bytes of our packed-word layout (8 B/cell each way + the tile faces), which move less
    roof = {"bound": "l2" if l2_resident else "hbm", "achieved": achieved_s, "peak": peak, "unit": "GB/s",
            "frac": (achieved_s / peak) if achieved_s else None, "traffic": traffic,
            "kernel": tag, "peak_source": peak_src,
            "algorithmic_bytes_per_cell_per_sweep": sbytes,
            "bytes_convention": "SURVEY.md 8(d): 13 B/cell SoA state read + written + tile halo, per outer round",
            "packed_word": {"bytes_per_cell_per_sweep": bpc, "achieved": achieved,
                            "frac": (achieved / peak) if achieved else None,
                            "note": "our layout: one 8 B packed word (t | n | s) read + written + tile faces"},
            "resident_note": ("the tiles stay in shared memory across sweeps: per sweep only their boundary lines "
                              "(0.25 B/cell) cross L2, so the byte roofline is nominal; the kernel is bound by the "
                              "issue rate and the grid barriers") if resident else None,
            "cells_per_sweep": n_local,
            "mean_sweep_ms": mean_sweep * 1e3, "sweeps_per_step": launches / args.steps,
            "kernel_launches_per_sweep": round(kl_per_sweep, 2),
            "kernel_share_of_step": ks / elapsed if elapsed else None}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "%s: %s" % (args.config, cfg["note"]), "dims": list(dims), "T": cfg["T"],
                       "beta": cfg["beta"], "h": cfg["h"], "rule": ["heatbath", "metropolis"][cfg["rule"]],
                       "tile": list(tile), "rounds_per_tile_visit": args.rounds or cfg.get("opts", {}).get("rounds_per_launch", aca.DEFAULT_ROUNDS),
                       "sweep": ("checkerboard: 2 grid-barrier phases per outer round inside one cooperative launch"
                                 if resident else "checkerboard: 2 kernel launches per outer round (tile colours 0, 1)"),
                       "parallelism": "row strips x %d" % world if ndim == 2 else "z slabs x %d" % world,
                       "halo_transport": (("cuda-ipc push" if args.transport == "ipc" else "nccl exchange")
                                          if world > 1 else "none (one shard)"),
                       "l2": ("state %.1f MB per GPU: L2-resident (roofline against measured L2 bandwidth)" %
                              (state_bytes / 1e6)) if l2_resident else
                             ("state %.2f GB per GPU >> 126 MB L2 (no flush needed)" % (state_bytes / 1e9)),
                       "shards": args.shards, "rows_div": args.rows_div,
                       "event_hash": not args.no_hash},
            "roofline": roof,
            "roofline_issue": issue_roofline(args.config),
            "firing_fraction": fired / tested if tested else None,
            "a10": {"early_reject": int(opts.get("early_reject", 0)), "class_book": int(opts.get("class_book", 0)),
                    "class_wmax": opts.get("class_wmax"),
                    "tile_visits_early_per_step": v_early // args.steps,
                    "tile_visits_plain_per_step": v_plain // args.steps},
            "arrivals_per_cell_per_sweep": (fired / launches / n_local) if launches else None,
            "gpu_launches": int(kl + 2 * args.steps),
            "clocks": clk}

    # end-to-end through the public API with host buffers: every step copies its initial spins
    # host -> device and its final spins device -> host (pinned buffers). The copies are
    # pipelined with the simulation through the asynchronous spin I/O calls: step k+1's input
    # is staged while step k runs, and step k's output drains while step k+1 runs.
    if not args.no_e2e:
        import torch as _t
        # the config's own initial distribution (c5: all +1 but an i.i.d. 5 %)
        host_in = [_t.from_numpy(workloads.host_spins((n_local,), seed=7 + j, q_minus=cfg["init_q"])).pin_memory()
                   for j in range(2)]
        host_out = [_t.empty(n_local, dtype=_t.int8).pin_memory() for _ in range(2)]

        def e2e_steps(n, seed0):
            """n pipelined steps, the first one's input staged inside; returns the arrivals"""
            arr = 0
            aca.aca_stage_spins(sim.handle, host_in[0], 0)
            for k in range(n):
                sim.reset(seed0 + k)
                aca.aca_set_spins_staged(sim.handle, k % 2)
                if k + 1 < n:
                    aca.aca_stage_spins(sim.handle, host_in[(k + 1) % 2], (k + 1) % 2)
                sim.run_until(cfg["T"])
                arr += sim.stats()["arrivals"]
                aca.aca_get_spins_async(sim.handle, host_out[k % 2])
            aca.aca_sync(sim.handle)
            torch.cuda.synchronize()
            return arr

        # untimed warm-up of this leg's own calls (the staging buffers, the copy stream and the
        # pinned pages are first touched here, not inside the timed region)
        e2e_steps(min(args.warmup, 3), args.seed + args.steps)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_arr = e2e_steps(args.steps, args.seed)
        et = time.perf_counter() - t0
        if world > 1:
            et = adist.reduce_max(et)
            e_arr = adist.reduce_sum_int(e_arr)
        line["e2e"] = {"value": e_arr / et, "unit": UNIT, "h2d_bytes_per_step": int(n_local),
                       "d2h_bytes_per_step": int(n_local) + 8 * 13}

    if rank == 0 and world == 1 and not args.no_cpu:
        v, arr, dt, sample = oracle_sample(cfg)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                                "cpu": cpu_name(), "host_cores": os.cpu_count()}
    uuid = str(torch.cuda.get_device_properties(local).uuid)
    if world > 1:
        import torch.distributed as tdist
        uuids = [None] * world
        tdist.all_gather_object(uuids, uuid)
        line["config"]["device_uuids"] = uuids
    else:
        line["config"]["device_uuids"] = [uuid]
    if rank == 0:
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
