"""Asynchronous spin I/O (aca_stage_spins / aca_set_spins_staged / aca_get_spins_async /
aca_sync): a pipelined multi-step loop with alternating staging slots gives, step by step, the
same spins as the synchronous calls, and those equal the serial oracle started from the same
user-supplied spins."""
import numpy as np
import pytest
import torch

import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,opts", [((200, 136), {}), ((256, 192), {"shards": 2}), ((40, 36, 24), {})])
def test_pipelined_steps_equal_synchronous_and_oracle(aca, oracle_mod, dims, opts):
    T, beta = 3.0, (0.4406868 if len(dims) == 2 else 0.2216544)
    n = int(np.prod(dims))
    inputs = [torch.from_numpy(workloads.host_spins((n,), seed=11 + k)).pin_memory() for k in range(3)]
    outs = [torch.empty(n, dtype=torch.int8).pin_memory() for _ in range(3)]

    a = aca.Sim(dims, beta=beta, seed=5, **opts)
    aca.aca_stage_spins(a.handle, inputs[0], 0)
    for k in range(3):
        a.reset(5 + k)
        aca.aca_set_spins_staged(a.handle, k % 2)
        if k + 1 < 3:
            aca.aca_stage_spins(a.handle, inputs[k + 1], (k + 1) % 2)   # overlaps this step's run
        a.run_until(T)
        aca.aca_get_spins_async(a.handle, outs[k])
    aca.aca_sync(a.handle)

    b = aca.Sim(dims, beta=beta, seed=5, **opts)
    for k in range(3):
        b.reset(5 + k)
        aca.aca_set_spins(b.handle, inputs[k])
        b.run_until(T)
        ref = aca.aca_get_spins(b.handle)
        assert np.array_equal(outs[k].numpy(), ref), k
        o = oracle_mod.OracleSim(dims, beta=beta, seed=5 + k)
        o.set_spins(inputs[k].numpy().reshape(dims[::-1]))
        o.run_until(T)
        assert np.array_equal(ref.reshape(dims[::-1]), o.spins()), k


def test_async_io_argument_errors(aca):
    s = aca.Sim((64, 64), beta=0.3, seed=1)
    with pytest.raises(aca.AcaError):
        aca.aca_set_spins_staged(s.handle, 0)          # nothing staged yet
    with pytest.raises(aca.AcaError):
        aca.aca_stage_spins(s.handle, np.ones(10, np.int8), 0)   # wrong count
    with pytest.raises(aca.AcaError):
        aca.aca_stage_spins(s.handle, np.ones(64 * 64, np.int8), 2)   # bad slot
