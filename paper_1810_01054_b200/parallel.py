"""Multi-GPU plumbing: one process per GPU, torch.distributed for the process
group, NCCL over NVLink/NVSwitch on GPUs (gloo on CPU for tests).

The path shards by independent rollouts (a batch of controllers or designs): rank g owns
rollouts [g*B/G, (g+1)*B/G) and runs them with no per-step communication.  The one real
exchange step is the reduction of gradients of parameters SHARED by all rollouts (e.g. one
actuation schedule or one E field optimised against a batch of scenes): a single
all-reduce(sum) per backward.  Timing is the max over ranks of device-measured times.
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
