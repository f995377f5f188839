"""Host-side multi-process plumbing (torch.distributed): partition of the sharded axis,
ncclUniqueId distribution, max/sum reductions of timings and counters, gathering of
rank-local shards, and the CUDA-IPC handle exchange of the multi-process push mode. No
arithmetic of the method lives here; the halo traffic itself runs inside libaca.so (kernel
stores into the neighbours' mapped halos, or NCCL send/recv).
Works with the gloo backend on CPU tensors (tests) and with nccl on GPUs (bench)."""
import numpy as np
import torch
import torch.distributed as dist


def env_world():
    import os
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def partition(dims, world):
    """Rows (2-D) / planes (3-D) of the sharded axis owned by each rank: equal contiguous
    strips (row-strip / z-slab partition of configs 3 and 4)."""
    axis = len(dims) - 1
    n = int(dims[axis])
    if world < 1 or n % world != 0:
        raise ValueError("%d ranks do not divide the sharded axis of length %d" % (world, n))
    step = n // world
    return [(r * step, (r + 1) * step) for r in range(world)]


def _device():
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_bytes(payload, src=0, nbytes=128):
    """Share rank src's bytes (e.g. a 128-byte ncclUniqueId) with every rank."""
    t = torch.zeros(nbytes, dtype=torch.uint8, device=_device())
    if dist.get_rank() == src:
        t.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().numpy().tobytes())


def all_gather_bytes(payload):
    """Every rank's bytes (equal lengths), concatenated in rank order."""
    b = bytes(payload)
    t = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(_device())
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return b"".join(bytes(o.cpu().numpy().tobytes()) for o in out)


def ipc_connect(handle):
    """Multi-process push mode: exchange the CUDA-IPC blobs (aca_ipc_export) of all ranks and
    map the neighbours' halos and every rank's slot into this process (aca_ipc_import)."""
    import paper_cs_0502039_b200 as aca
    aca.aca_ipc_import(handle, all_gather_bytes(aca.aca_ipc_export(handle)))


def reduce_max(x):
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum_int(x):
    t = torch.tensor([int(x)], dtype=torch.int64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


def gather_shards(local, dims):
    """Assemble the global array (x fastest, sharded axis slowest) from rank-local shards."""
    world = dist.get_world_size()
    t = torch.as_tensor(np.ascontiguousarray(local).view(np.uint8)).to(_device())
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    full = np.concatenate([o.cpu().numpy() for o in out]).view(local.dtype)
    return full.reshape(tuple(dims)[::-1])
