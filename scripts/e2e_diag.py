"""c5 e2e diagnostic: per-step wall time and tile-path counts of device-initialised steps vs
steps whose spins come from the host (aca_set_spins_staged), as bench.py's e2e leg runs them."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_cs_0502039_b200 as aca
import workloads

C = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = workloads.config(C)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
opts = dict(init_q=cfg["init_q"], device=0, tile=tuple(cfg["tile"]), stream=stream.cuda_stream)
opts.update(cfg.get("opts", {}))
sim = aca.Sim(tuple(cfg["dims"]), lam=cfg["lam"], beta=cfg["beta"], J=cfg["J"], h=cfg["h"], rule=cfg["rule"], seed=1, **opts)
n = aca.aca_num_cells(sim.handle)
host_in = [torch.from_numpy(workloads.host_spins((n,), seed=7 + j, q_minus=cfg["init_q"])).pin_memory() for j in range(2)]
host_out = [torch.empty(n, dtype=torch.int8).pin_memory() for _ in range(2)]
def show(tag, t, st):
    print("%-8s %.1f ms  arrivals %.3e  early %d plain %d  kernel_s %.3f launches %d  ->%.3e/s" % (
        tag, t * 1e3, st["arrivals"], st["tile_visits_early"], st["tile_visits_plain"], st["kernel_seconds"], st["launches"], st["arrivals"] / t))
for k in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sim.reset(1 + k); sim.run_until(cfg["T"]); st = sim.stats()
    torch.cuda.synchronize(); show("dev", time.perf_counter() - t0, st)
for k in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    aca.aca_stage_spins(sim.handle, host_in[k % 2], k % 2)
    sim.reset(1 + k); aca.aca_set_spins_staged(sim.handle, k % 2)
    sim.run_until(cfg["T"]); st = sim.stats()
    aca.aca_get_spins_async(sim.handle, host_out[k % 2]); aca.aca_sync(sim.handle)
    torch.cuda.synchronize(); show("host", time.perf_counter() - t0, st)
for k in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sim.reset(1 + k); sim.set_spins(host_in[k % 2].numpy()) if hasattr(sim, "set_spins") else None
    sim.run_until(cfg["T"]); st = sim.stats()
    torch.cuda.synchronize(); show("setsp", time.perf_counter() - t0, st)
