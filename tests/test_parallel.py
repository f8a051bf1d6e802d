"""Host-side multi-rank logic on CPU: world_size 2 with the gloo backend (the GPU path uses
the same code with NCCL).  No CUDA is needed."""
import os
import socket

import numpy as np
import pytest

from paper_1810_01054_b200 import parallel, scenes


@pytest.mark.parametrize("n,world", [(64, 2), (64, 8), (7, 3), (2, 4), (0, 2), (1000, 7)])
def test_shard_range_partition(n, world):
    seen = []
    sizes = []
    for r in range(world):
        lo, hi = parallel.shard_range(n, world, r)
        seen += list(range(lo, hi))
        sizes.append(hi - lo)
    assert seen == list(range(n))
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist
    d = parallel.init_from_env("gloo")
    sc = scenes.quadruped_3d(batch=5, steps=4, e_scale=True)
    mine = parallel.shard_scene(sc, d)
    # per-rollout actuation gradients (stand-in values: rollout index + 1)
    lo, hi = mine.meta["shard"]
    da_local = np.stack([np.full((4, sc.n_act, 3), r + 1.0, np.float32) for r in range(lo, hi)])
    tot = parallel.shared_actuation_grad(da_local, d)
    mx = parallel.max_over_ranks(10.0 * (rank + 1), d)
    q.put((rank, lo, hi, mine.batch, float(tot[0, 0, 0]), mx,
           float(np.abs(mine.x - sc.x[lo:hi]).max())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_rollouts_and_shared_grad():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, b0, t0, m0, e0), (r1, lo1, hi1, b1, t1, m1, e1) = res
    assert (lo0, hi0, lo1, hi1) == (0, 3, 3, 5) and b0 == 3 and b1 == 2
    # shared-parameter gradient: sum over all 5 rollouts of (r + 1) = 15 on every rank
    assert t0 == t1 == 15.0
    assert m0 == m1 == 20.0
    assert e0 == 0.0 and e1 == 0.0


# ---- slab sharding (SURVEY 8e, configs[4]) -------------------------------------------------

@pytest.mark.parametrize("dim,res,G,halo", [(3, 64, 2, 1), (3, 64, 3, 1), (3, 256, 8, 1), (2, 128, 4, 1),
                                            (3, 128, 4, 2), (2, 64, 3, 1)])
def test_slab_partition_properties(dim, res, G, halo):
    """Block-aligned, covering, every slab >= 2*halo blocks wide (libmpm's window rule),
    balanced to within one block-plane of particles, membership disjoint and complete."""
    rng = np.random.default_rng(dim * 100 + G)
    n = 20000
    x = rng.uniform(0.1, 0.7, (n, dim)).astype(np.float32)
    x[:, 0] = (0.15 + 0.6 * rng.beta(2.0, 5.0, n)).astype(np.float32)  # skewed in x
    b = parallel.slab_partition(x, res, dim, G, halo)
    BB = parallel.block_size(dim)
    assert b[0][0] == 0 and b[-1][1] == res and len(b) == G
    for (lo, hi), (lo2, _) in zip(b, b[1:] + [(res, None)]):
        assert lo % BB == 0 and hi % BB == 0 and hi == lo2
        assert hi - lo >= 2 * halo * BB
    idx = [parallel.slab_members(x, res, lo, hi) for lo, hi in b]
    allidx = np.sort(np.concatenate(idx))
    np.testing.assert_array_equal(allidx, np.arange(n))
    bx = parallel.base_x(x, res)
    plane = np.bincount(np.clip(bx, 0, res - 1) // BB, minlength=res // BB).max()
    counts = [len(i) for i in idx]
    if all(hi - lo > 2 * halo * BB for lo, hi in b):  # the width rule did not bind
        assert max(counts) - n / G <= plane + 1, counts


def test_slab_partition_infeasible():
    x = np.full((10, 3), 0.5, np.float32)
    with pytest.raises(ValueError):
        parallel.slab_partition(x, 32, 3, 5, 1)  # 8 block-planes cannot hold 5 slabs of 2


def _slab_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist
    d = parallel.init_from_env("gloo")
    sc = scenes.quadruped_3d(steps=4)
    bounds = parallel.slab_partition(sc.x[0], sc.res, sc.dim, d.world)
    lo, hi = bounds[d.rank]
    mine, idx = parallel.shard_slab(sc, lo, hi)
    cnt = torch.tensor([mine.n], dtype=torch.int64)
    dist.all_reduce(cnt)
    # every rank derived the same partition
    allb = [None] * world
    dist.all_gather_object(allb, bounds)
    owned = torch.zeros(sc.n, dtype=torch.int64)
    owned[torch.as_tensor(idx)] = 1
    dist.all_reduce(owned)
    q.put((rank, lo, hi, int(cnt.item()), sc.n, all(b == bounds for b in allb),
           int(owned.min()), int(owned.max()), float(np.abs(mine.x[0] - sc.x[0][idx]).max())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_slab_partition_agrees():
    """Each rank computes its slab and particles from the shared scene; the union over ranks
    owns every particle exactly once and all ranks derived the same slab bounds."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_slab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, c0, n0, same0, mn0, mx0, e0), (r1, lo1, hi1, c1, n1, same1, mn1, mx1, e1) = res
    assert lo0 == 0 and hi0 == lo1 and hi1 == 64
    assert c0 == c1 == n0 == n1
    assert same0 and same1 and mn0 == mx0 == 1 and e0 == 0.0 and e1 == 0.0


def _comm_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist
    from paper_1810_01054_b200 import mpm
    d = parallel.init_from_env("gloo")
    if rank == 0:
        mpm.comm_unique_id = lambda: bytes(np.random.default_rng(1234).integers(0, 256, 128, dtype=np.uint8))
    else:  # only rank 0 may create the id; the others must receive it
        def _no(*_):
            raise AssertionError("comm_unique_id called on a non-zero rank")
        mpm.comm_unique_id = _no

    class Recorder:  # stands in for an MPM context: records what comm_init receives
        def comm_init(self, r, w, uid):
            self.got = (r, w, uid)

    rec = Recorder()
    parallel.init_slab_comm(rec, d)
    q.put((rank, rec.got[0], rec.got[1], rec.got[2].hex()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_slab_comm_handshake():
    """init_slab_comm: rank 0 creates the NCCL id, torch.distributed broadcasts it, every rank
    joins with (its rank, world, the same id)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_comm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, w0, u0), (r1, a1, w1, u1) = res
    assert (a0, a1, w0, w1) == (0, 1, 2, 2) and u0 == u1 and len(u0) == 256
