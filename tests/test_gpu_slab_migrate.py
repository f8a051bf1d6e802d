"""Migrating slab mode ("halo exchange of ghost grid nodes and migrating particles";
include/mpm.h mpm_set_slab_migrating): ownership by base_x at EVERY step, the particles that
leave a slab after G2P are sent to the neighbour and appended to its next state, and the
backward returns the adjoints along the same paths (reverse migration).  The grid windows are
summed as in the Lagrangian slab mode.

Multi-rank runs are emulated on ONE GPU: mpm_group_forward / mpm_group_backward (the same
kernels, device copies in place of the exchanges, host-sequenced), and -- across processes --
two processes sharing cuda:0 that exchange through mpm_set_transport with gloo
(host-staged: no kernel waits on another).  Every check is against the fp64 oracle of the WHOLE
body: the sharded run must compute the unsharded step, for a body that travels across several
slab boundaries (the paper's walker runs for "maximum distance")."""
import os

import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm, parallel, scenes
from tests.helpers import assert_grads, oracle_cfg, oracle_params, oracle_state

pytestmark = pytest.mark.gpu


def _walker(dim):
    """A walker-like actuated body with random F0 / C0 running in +x across two slab
    boundaries (slabs below): 2D 128^2, 3D 64^3."""
    if dim == 2:
        sc = scenes.tiny(2, seed=21, res=128, n_cells=(20, 8), center=(36, 40), steps=240, v0=(20.0, 0.0), K=3,
                         s=40.0, gravity=(0.0, -2.0))
        return sc, [(0, 48), (48, 64), (64, 128)]
    sc = scenes.tiny(3, seed=22, res=64, n_cells=(10, 4, 4), center=(17, 20, 30), steps=220, v0=(14.0, 0.0, 0.0),
                     K=3, s=40.0, gravity=(0.0, -2.0, 0.0))
    return sc, [(0, 24), (24, 32), (32, 64)]


def _oracle_run(sc, T, seed):
    cfg = oracle_cfg(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    w = np.random.default_rng(seed).standard_normal(traj[T].shape)
    g = oracle.backward(cfg, traj, m, vol, E, nu, aid, act[:T], w)
    return traj, w, g


def _sims(sc, T, bounds, cap_frac=1.0, mig_cap=0, halo=1):
    sims = []
    for lo, hi in bounds:
        cfg = mpm.Config.from_scene(sc, max_steps=T)
        cfg.n_particles = max(64, int(cap_frac * sc.n))  # storage capacity of the slab
        sim = mpm.MPM(cfg)
        sim.set_slab_migrating(lo, hi, halo, sc.n, mig_cap)
        sim.set_scene(sc)  # whole-body arrays; each slab keeps what it owns
        sims.append(sim)
    return sims


def _sum_state(sims, t):
    out = None
    for s in sims:
        st = s.get_state(t)
        out = [a.astype(np.float64) for a in st] if out is None else [o + a for o, a in zip(out, st)]
    return out


def _check(sc, T, bounds, sims, orc, group=True):
    traj, w, (g0, gE, gnu, ga) = orc
    d = sc.dim
    # every particle is owned by exactly one slab at t = 0 and at T
    x0 = _sum_state(sims, 0)[0]
    np.testing.assert_allclose(x0, sc.x[0], rtol=0, atol=0)
    x, v, F, Cm = _sum_state(sims, T)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    vmax = max(np.abs(ov).max(), 1e-6)
    for k, a, b, scale in (("x", x, ox, 1.0), ("v", v, ov, vmax), ("F", F, oF, np.abs(oF).max()),
                           ("C", Cm, oC, 4 * sc.res * vmax)):
        assert np.abs(a - b).max() / scale < 1e-4, (k, bounds)
    wx, wv, wC, wF = oracle.unpack(w, d)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    if group:
        n = len(sims)
        mpm.group_backward(sims, [f32(wx)] * n, [f32(wv)] * n, [f32(wF)] * n, [f32(wC)] * n)
    grads = [s.grad() for s in sims]
    full = {k: sum(g[k].astype(np.float64) for g in grads) for k in ("dx0", "dv0", "dF0", "dC0")}
    for g in grads[1:]:  # whole-body sums on every slab
        for k in ("dE", "dnu", "da"):
            np.testing.assert_array_equal(g[k], grads[0][k])
    gx, gv, gC, gF = oracle.unpack(g0, d)
    assert_grads([("dx0", full["dx0"], gx), ("dv0", full["dv0"], gv), ("dF0", full["dF0"], gF),
                  ("dC0", full["dC0"], gC), ("dE", grads[0]["dE"], gE), ("dnu", grads[0]["dnu"], gnu),
                  ("da", grads[0]["da"][0, :T], ga)], ctx=bounds)


@pytest.mark.parametrize("dim", [2, 3])
def test_migrating_walker_crosses_two_boundaries(dim):
    """A body running across two slab boundaries over 220-240 steps, 3 slabs: particles
    migrate 0 -> 1 and 1 -> 2 (asserted from the oracle trajectory), whole-body state and every
    gradient family (element-wise) vs the oracle."""
    sc, bounds = _walker(dim)
    T = sc.steps
    orc = _oracle_run(sc, T, 31 + dim)
    bx0 = np.floor(sc.x[0][:, 0].astype(np.float32) * np.float32(sc.res) - np.float32(0.5))
    bxT = np.floor(orc[0][T][:, 0] * sc.res - 0.5)
    for _, hi in bounds[:-1]:
        assert np.sum((bx0 < hi) & (bxT >= hi)) > 0, ("no particle crosses", hi)
    sims = _sims(sc, T, bounds)
    mpm.group_forward(sims, T)
    _check(sc, T, bounds, sims, orc)
    for s in sims:
        s.close()


def test_migrating_matches_lagrangian_and_plain():
    """The migrating split of a small body that crosses one boundary equals the unsharded run
    up to fp32 summation order (and both match the oracle)."""
    sc = scenes.tiny(3, seed=23, res=32, n_cells=(6, 3, 3), center=(9, 12, 12), steps=60, v0=(14.0, 0.0, 0.0), K=2,
                     s=30.0)
    T = sc.steps
    bounds = [(0, 16), (16, 32)]
    orc = _oracle_run(sc, T, 41)
    sims = _sims(sc, T, bounds, cap_frac=1.0)
    mpm.group_forward(sims, T)
    _check(sc, T, bounds, sims, orc)


def test_migrate_capacity_errors():
    """mig_cap too small for the leavers of a step latches MPM_ERR_MIGRATE; a capacity below the
    slab's t = 0 members is refused at set_state."""
    sc, bounds = _walker(2)
    T = 40
    sims = _sims(sc, T, bounds, mig_cap=1)
    with pytest.raises(mpm.MPMError) as e:
        mpm.group_forward(sims, T)
    assert e.value.status == "MPM_ERR_MIGRATE"
    cfg = mpm.Config.from_scene(sc, max_steps=T)
    cfg.n_particles = 8
    sim = mpm.MPM(cfg)
    sim.set_slab_migrating(*bounds[0], 1, sc.n, 0)
    with pytest.raises(mpm.MPMError) as e:
        sim.set_scene(sc)
    assert e.value.status == "MPM_ERR_MIGRATE"


# ---- two processes on one GPU, host-staged exchanges through gloo --------------------------------
def _rank_main(rank, world, port, q, mode="migrate"):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sc = scenes.quadruped_3d(steps=40)
        T = 40
        bx = np.floor(sc.x[0][:, 0] * sc.res - 0.5)
        cut = 32  # two slabs of the 64^3 quadruped (block-aligned)
        bounds = [(0, cut), (cut, sc.res)]
        lo, hi = bounds[rank]
        idx = None
        if mode == "migrate":
            cfg = mpm.Config.from_scene(sc, max_steps=T)
            cfg.n_particles = int(0.9 * sc.n)
            sim = mpm.MPM(cfg)
            sim.set_slab_migrating(lo, hi, 1, sc.n, 0)
        else:  # Lagrangian ownership, fused forward (windows of grid t+1 summed between launches)
            sc_full = sc
            sc, idx = parallel.shard_slab(sc_full, lo, hi)
            sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, fuse_g2p2g=1))
            sim.set_slab(lo, hi, 1)
            sim.set_profiling(True)

        def xchg(kind, sl, sr, rl, rr):
            if kind == "reduce":
                t = torch.from_numpy(sl)
                dist.all_reduce(t)
                return
            reqs = []
            if sl is not None:
                reqs.append(dist.isend(torch.from_numpy(sl.copy()), rank - 1))
                reqs.append(dist.irecv(torch.from_numpy(rl), rank - 1))
            if sr is not None:
                reqs.append(dist.isend(torch.from_numpy(sr.copy()), rank + 1))
                reqs.append(dist.irecv(torch.from_numpy(rr), rank + 1))
            for r in reqs:
                r.wait()

        sim.set_transport(xchg)
        sim.set_scene(sc)
        sim.forward(T)
        if idx is not None:
            pf = sim.profile()
            assert pf["p2g"][1] == 1 and pf["g2p2g"][1] == T and pf["band_pack"][1] == T, pf
        st = [a.copy() for a in sim.get_state(T)]
        rng = np.random.default_rng(51)
        w = rng.standard_normal((scenes.quadruped_3d(steps=40).n, oracle.S_of(3)))
        if idx is not None:
            w = w[idx]
        wx, wv, wC, wF = oracle.unpack(w, 3)
        f32 = lambda a: np.ascontiguousarray(a, np.float32)
        sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
        g = sim.grad()
        q.put((rank, st, {k: np.asarray(v).copy() for k, v in g.items()}, int(np.sum(bx >= cut)), idx))
        sim.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, "error", traceback.format_exc(), None, None))


@pytest.mark.parametrize("mode", ["migrate", "lagrangian_fused"])
def test_two_processes_gloo_transport_vs_oracle(mode):
    """configs[2]'s quadruped (29,952 particles) split at x = 32 between two PROCESSES on cuda:0,
    exchanging through gloo (mpm_set_transport); summed / gathered state and gradients vs the
    whole-body oracle -- the collective call order of forward / get_state / backward / grad and
    the gradient reductions across processes.  migrate: Eulerian ownership with migrants and
    reverse-migrated adjoints; lagrangian_fused: fixed ownership with the fused forward (the
    windows of grid t+1 summed between two G2P2G launches)."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=120)
    for r in res.values():
        assert r[1] != "error", r[2]
    sc = scenes.quadruped_3d(steps=40)
    T = 40
    traj, w, (g0, gE, gnu, ga) = _oracle_run(sc, T, 51)
    if mode == "migrate":
        st = [res[0][1][i].astype(np.float64) + res[1][1][i] for i in range(4)]
        g = {k: res[0][2][k].astype(np.float64) + res[1][2][k] for k in ("dx0", "dv0", "dF0", "dC0", "dE", "dnu")}
    else:  # each process holds its shard (parallel.shard_slab indices)
        st = [np.zeros((sc.n,) + a.shape[1:]) for a in res[0][1]]
        g = {k: np.zeros((sc.n,) + np.asarray(res[0][2][k]).shape[1:]) for k in ("dx0", "dv0", "dF0", "dC0", "dE", "dnu")}
        for r in (0, 1):
            idx = res[r][4]
            for i in range(4):
                st[i][idx] = res[r][1][i]
            for k in g:
                g[k][idx] = res[r][2][k]
    ox, ov, oC, oF = oracle.unpack(traj[T], 3)
    vmax = np.abs(ov).max()
    for k, a, b, scale in (("x", st[0], ox, 1.0), ("v", st[1], ov, vmax), ("F", st[2], oF, np.abs(oF).max()),
                           ("C", st[3], oC, 4 * sc.res * vmax)):
        assert np.abs(a - b).max() / scale < 1e-4, k
    if mode == "migrate":
        np.testing.assert_array_equal(res[0][2]["dE"], res[1][2]["dE"])
        gE_gpu, gnu_gpu = res[0][2]["dE"], res[0][2]["dnu"]
    else:
        gE_gpu, gnu_gpu = g["dE"], g["dnu"]
    np.testing.assert_array_equal(res[0][2]["da"], res[1][2]["da"])  # the shared actuation gradient
    gx, gv, gC, gF = oracle.unpack(g0, 3)
    assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF), ("dC0", g["dC0"], gC),
                  ("dE", gE_gpu, gE), ("dnu", gnu_gpu, gnu), ("da", res[0][2]["da"][0, :T], ga)], ctx=mode)
    assert 0 < res[0][3] < sc.n  # both slabs own particles
