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
