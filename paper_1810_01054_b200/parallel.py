"""Multi-GPU plumbing: one process per GPU, torch.distributed for the process
group, NCCL over NVLink/NVSwitch on GPUs (gloo on CPU for tests).

Batch sharding: rank g owns rollouts [g*B/G, (g+1)*B/G) and runs them with no per-step
communication.  The one real exchange step is the reduction of gradients of parameters
SHARED by all rollouts (e.g. one actuation schedule or one E field optimised against a batch
of scenes): a single all-reduce(sum) per backward.

Slab sharding (one large rollout, configs[4] "8M particles slab-sharded"): rank g owns the
particles whose base_x lies in its x-slab [x_lo, x_hi) at t = 0; libmpm sums the grid windows
around each slab boundary with its x-neighbours (NCCL send/recv, include/mpm.h "slab mode").
This module holds the host side: a particle-count-balanced partition, slab membership, and
the NCCL-id handshake.  Timing is the max over ranks of device-measured times.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass
class Dist:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    group: object = None

    @property
    def active(self) -> bool:
        return self.world > 1


def init_from_env(backend: str | None = None) -> Dist:
    """Read RANK / WORLD_SIZE / LOCAL_RANK (torchrun) and initialise the default process
    group when WORLD_SIZE > 1.  backend defaults to nccl with CUDA, gloo otherwise."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world > 1:
        import torch
        import torch.distributed as dist
        if not dist.is_initialized():
            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            kw = {}
            if backend == "nccl":
                torch.cuda.set_device(local)
                kw["device_id"] = torch.device("cuda", local)
            dist.init_process_group(backend, **kw)
    return Dist(rank, world, local)


def shard_range(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced, disjoint shard [lo, hi) of n_items for `rank` (sizes differ by
    at most one; every item is owned by exactly one rank)."""
    if world < 1 or not (0 <= rank < world) or n_items < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def allreduce_sum_(t, d: Dist):
    """In-place sum over ranks of a torch tensor (shared-parameter gradients)."""
    if d.active:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def max_over_ranks(x: float, d: Dist, device=None) -> float:
    """Max over ranks of a scalar (device timings are reported as the slowest rank)."""
    if not d.active:
        return float(x)
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "gloo":
        device = None  # host tensors for gloo
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shared_actuation_grad(da_local: np.ndarray, d: Dist, device=None) -> np.ndarray:
    """Gradient w.r.t. ONE actuation schedule shared by all rollouts of all ranks:
    da_local [B_local][T][K][dim] (per-rollout gradients from mpm_grad) -> sum over the
    local rollouts, then all-reduce(sum) over ranks -> [T][K][dim]."""
    import torch
    t = torch.as_tensor(np.ascontiguousarray(da_local.sum(axis=0), np.float32), device=device)
    allreduce_sum_(t, d)
    return t.cpu().numpy()


def shard_scene(sc, d: Dist):
    """The rollouts of a batched scene owned by this rank (a Scene with batch = shard)."""
    import copy
    lo, hi = shard_range(sc.batch, d.world, d.rank)
    out = copy.copy(sc)
    for name in ("x", "v", "F", "C", "mass", "vol", "E", "nu", "actuator_id", "act"):
        setattr(out, name, np.ascontiguousarray(getattr(sc, name)[lo:hi]))
    out.meta = dict(sc.meta, shard=(lo, hi))
    return out


def block_size(dim: int) -> int:
    """Grid-block edge in nodes (libmpm: 4 in 3D, 8 in 2D)."""
    return 4 if dim == 3 else 8


def base_x(x: np.ndarray, res: int) -> np.ndarray:
    """floor(x * res - 0.5) of the x coordinate, decided in fp32 like the binning (R17)."""
    xs = np.asarray(x, np.float32)[..., 0]
    return np.floor(xs * np.float32(res) - np.float32(0.5)).astype(np.int64)


def slab_partition(x: np.ndarray, res: int, dim: int, world: int, halo: int = 1) -> list[tuple[int, int]]:
    """Split [0, res) node planes into `world` x-slabs [x_lo, x_hi) at block boundaries with
    balanced particle counts (by base_x at t = 0), every slab at least 2*halo blocks wide
    (libmpm's window constraint).  Deterministic: every rank computes the same answer."""
    BB = block_size(dim)
    nbp = res // BB
    if world < 1:
        raise ValueError("world >= 1")
    if world == 1:
        return [(0, res)]
    w = 2 * halo
    if nbp < world * w:
        raise ValueError(f"{world} slabs of >= {w} block-planes do not fit in {nbp}")
    bx = np.clip(base_x(x, res), 0, res - 1) // BB
    cum = np.cumsum(np.bincount(bx, minlength=nbp))  # particles with block-plane <= k
    n = cum[-1]
    b = [0] + [int(np.searchsorted(cum, g * n / world, side="left")) + 1 for g in range(1, world)] + [nbp]
    for g in range(1, world):  # widths >= w, forward then backward
        b[g] = max(b[g], b[g - 1] + w)
    for g in range(world - 1, 0, -1):
        b[g] = min(b[g], b[g + 1] - w)
    if any(b[g + 1] - b[g] < w for g in range(world)) or b[0] != 0:
        raise ValueError("no feasible slab partition")
    return [(b[g] * BB, b[g + 1] * BB) for g in range(world)]


def slab_members(x: np.ndarray, res: int, lo: int, hi: int) -> np.ndarray:
    """Indices of the particles owned by slab [lo, hi) (base_x in [lo, hi); the first slab
    also takes base_x < 0 and the last base_x >= res, which the domain check rejects)."""
    bx = base_x(x, res)
    sel = (bx >= lo) & (bx < hi)
    if lo == 0:
        sel |= bx < 0
    if hi == res:
        sel |= bx >= res
    return np.nonzero(sel)[0]


def shard_slab(sc, lo: int, hi: int):
    """The particles of a single-rollout scene owned by slab [lo, hi): (Scene, user indices)."""
    import copy
    if sc.batch != 1:
        raise ValueError("slab sharding takes one rollout")
    idx = slab_members(sc.x[0], sc.res, lo, hi)
    out = copy.copy(sc)
    for name in ("x", "v", "F", "C", "mass", "vol", "E", "nu", "actuator_id"):
        setattr(out, name, np.ascontiguousarray(getattr(sc, name)[:, idx]))
    out.meta = dict(sc.meta, slab=(lo, hi))
    return out, idx


def gloo_transport(d: Dist):
    """A host-staged slab-exchange callback for `MPM.set_transport` over the default
    torch.distributed process group (e.g. gloo, ranks sharing one GPU): neighbour windows /
    migrants / adjoints with isend/irecv to rank -+ 1, the gradient sums with all_reduce."""
    import torch
    import torch.distributed as dist

    def xchg(kind, sl, sr, rl, rr):
        if kind == "reduce":
            t = torch.from_numpy(sl)
            dist.all_reduce(t)
            return
        reqs = []
        if sl is not None:
            reqs.append(dist.isend(torch.from_numpy(sl.copy()), d.rank - 1))
            reqs.append(dist.irecv(torch.from_numpy(rl), d.rank - 1))
        if sr is not None:
            reqs.append(dist.isend(torch.from_numpy(sr.copy()), d.rank + 1))
            reqs.append(dist.irecv(torch.from_numpy(rr), d.rank + 1))
        for r in reqs:
            r.wait()
    return xchg


def init_slab_comm(sim, d: Dist):
    """NCCL communicator of the slab ranks: rank 0 creates the id, torch.distributed
    broadcasts it, every rank joins (collective)."""
    from . import mpm
    uid = mpm.comm_unique_id() if d.rank == 0 else None
    if d.active:
        import torch.distributed as dist
        box = [uid]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]
    sim.comm_init(d.rank, d.world, uid)
