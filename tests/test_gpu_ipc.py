"""Multi-process push mode (CUDA IPC) on one GPU: two processes each own a strip / slab
(world 2, halo_mode 0), exchange their IPC blobs over gloo, and their tile kernels store
boundary rows straight into the other process's halo buffers (PAPER.md:741-750, 979-989:
neighbours read the boundary copies without waiting for each other; the conservative
firing test makes any interleaving exact). The assembled lattice must equal the serial
oracle bit for bit, after several successive runs (epoch barrier + termination slots).

The two processes never wait for each other inside a kernel (the host polls small slots),
so sharing one GPU by time slicing is safe."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, dims, Ts, kw):
    import torch
    import torch.distributed as dist

    import paper_cs_0502039_b200 as aca
    from paper_cs_0502039_b200 import dist as adist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        sim = aca.Sim(dims, world=world, rank=rank, device=0, **kw)
        adist.ipc_connect(sim.handle)
        st0 = sim.stats()            # right after create: the halos hold the neighbours' P5 rows
        for T in Ts:
            sim.run_until(T)
        st = sim.stats()
        q.put((rank, sim.spins().copy(), sim.times().copy(), sim.counters().copy(), st["cells_fired"], None,
               {k: st0[k] for k in ("bond_sum", "class_hist")}, {k: st[k] for k in ("bond_sum", "class_hist")}))
        dist.barrier()   # keep the mappings alive until every rank has read its result
        sim.close()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, None, None, 0, repr(e), None, None))
    finally:
        dist.destroy_process_group()


def _run_world(dims, Ts, world=2, **kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, dims, Ts, kw)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in res:
        assert r[5] is None, r[5]
    cat = lambda i: np.concatenate([r[i].reshape(-1) for r in res]).reshape(tuple(dims)[::-1])
    _run_world.stats = [(r[6], r[7]) for r in res]   # per rank: (after create, after the runs)
    return cat(1), cat(2), cat(3), sum(r[4] for r in res)


@pytest.mark.parametrize("dims,beta,tile", [((256, 192), 0.4406868, (64, 64)),
                                            ((200, 136), 0.4406868, (64, 64)),
                                            ((32, 24, 16), 0.2216544, (16, 16, 16))])
def test_ipc_push_two_processes(oracle_mod, dims, beta, tile):
    Ts = [1.0, 3.0, 5.0]
    s, t, n, fired = _run_world(dims, Ts, beta=beta, seed=61, tile=tile)
    o = oracle_mod.OracleSim(dims, lam=1.0, beta=beta, J=1.0, h=0.0, rule=0, seed=61, init_q=0.5)
    # statistics read the neighbours' boundary rows: right after create (their P5 rows) and after
    # the runs (the snapshot taken when every rank was done); the bond sums add up exactly
    assert sum(a["bond_sum"] for a, _ in _run_world.stats) == o.stats()["bond_sum"]
    for T in Ts:
        o.run_until(T)
    assert sum(b["bond_sum"] for _, b in _run_world.stats) == o.stats()["bond_sum"]
    assert np.array_equal(s, o.spins())
    assert np.array_equal(t, o.times())
    assert np.array_equal(n, o.counters())
    assert fired == o.stats()["arrivals"]


def test_ipc_push_four_processes_metropolis(oracle_mod):
    dims = (128, 128)
    s, t, n, fired = _run_world(dims, [4.0], world=4, beta=0.5, rule=1, seed=7, tile=(32, 32))
    o = oracle_mod.OracleSim(dims, lam=1.0, beta=0.5, J=1.0, h=0.0, rule=1, seed=7, init_q=0.5)
    o.run_until(4.0)
    assert np.array_equal(t, o.times()) and np.array_equal(s, o.spins()) and np.array_equal(n, o.counters())
    assert fired == o.stats()["arrivals"]
