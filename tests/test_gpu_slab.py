"""Slab mode (configs[4] "8M particles slab-sharded"): one rollout split into
x-slabs, each simulated by its own context, whose grid windows around every slab boundary
are summed between neighbours after P2G (forward) and after G2P^T (backward).

The multi-rank run is emulated on ONE GPU by mpm_group_forward / mpm_group_backward: the
same pack / exchange / unpack kernels as the NCCL path, with device copies standing in for
the NCCL send/recv, sequenced by the host (no kernel waits on another).  Every check is
against the fp64 oracle of the WHOLE body (a sharded run must compute the unsharded step)."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm, parallel, scenes
from tests.helpers import assert_grads, oracle_cfg, rel_err

pytestmark = pytest.mark.gpu


def _slab_sims(sc, T, G, halo=1, fuse=0):
    bounds = parallel.slab_partition(sc.x[0], sc.res, sc.dim, G, halo)
    sims, idxs = [], []
    for lo, hi in bounds:
        s2, idx = parallel.shard_slab(sc, lo, hi)
        sim = mpm.MPM(mpm.Config.from_scene(s2, max_steps=T, fuse_g2p2g=fuse))
        sim.set_slab(lo, hi, halo)
        sim.set_scene(s2)
        sims.append(sim)
        idxs.append(idx)
    assert sum(len(i) for i in idxs) == sc.n
    return sims, idxs, bounds


def _gather_state(sims, idxs, sc, t):
    d, n = sc.dim, sc.n
    out = [np.empty((n, d), np.float32), np.empty((n, d), np.float32),
           np.empty((n, d, d), np.float32), np.empty((n, d, d), np.float32)]
    for sim, idx in zip(sims, idxs):
        for o, a in zip(out, sim.get_state(t)):
            o[idx] = a
    return out


def _oracle(sc, T, seed):
    cfg = oracle_cfg(sc)
    st = oracle.pack(sc.x[0], sc.v[0], sc.C[0], sc.F[0])
    prm = [a[0].astype(np.float64) for a in (sc.mass, sc.vol, sc.E, sc.nu)]
    aid, act = sc.actuator_id[0], sc.act[0].astype(np.float64)[:T]
    traj = oracle.forward(cfg, st, *prm, aid, act, T)
    w = np.random.default_rng(seed).standard_normal(traj[T].shape)
    g = oracle.backward(cfg, traj, *prm, aid, act, w)
    return traj, w, g


def _check_slab_run(sc, T, G, halo=1, seed=5, tol=1e-3, orc=None, fuse=0):
    sims, idxs, bounds = _slab_sims(sc, T, G, halo, fuse)
    if fuse:
        for sim in sims:
            sim.set_profiling(True)
    mpm.group_forward(sims, T)
    if fuse:  # the fused forward really ran: one unfused P2G, then G2P2G with window sums between
        for sim in sims:
            pf = sim.profile()
            assert pf["p2g"][1] == 1 and pf["g2p2g"][1] == T and pf["band_pack"][1] == T, pf
    x, v, F, Cm = _gather_state(sims, idxs, sc, T)
    traj, w, (g0, gE, gnu, ga) = orc if orc is not None else _oracle(sc, T, seed)
    ox, ov, oC, oF = oracle.unpack(traj[T], sc.dim)
    for k, a, b in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC)):
        assert rel_err(a, b) < tol, (k, rel_err(a, b), bounds)
    wx, wv, wC, wF = oracle.unpack(w, sc.dim)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    mpm.group_backward(sims, [f32(wx[i]) for i in idxs], [f32(wv[i]) for i in idxs],
                       [f32(wF[i]) for i in idxs], [f32(wC[i]) for i in idxs])
    d, n = sc.dim, sc.n
    full = dict(dx0=np.empty((n, d)), dv0=np.empty((n, d)), dF0=np.empty((n, d, d)),
                dC0=np.empty((n, d, d)), dE=np.empty(n), dnu=np.empty(n))
    das = []
    for sim, idx in zip(sims, idxs):
        g = sim.grad()
        for k in full:
            full[k][idx] = g[k]
        das.append(g["da"][0, :T])
    for a in das[1:]:  # the shared actuation gradient is the same sum on every slab
        np.testing.assert_array_equal(a, das[0])
    gx, gv, gC, gF = oracle.unpack(g0, sc.dim)
    pairs = [(k, full[k], b) for k, b in (("dx0", gx), ("dv0", gv), ("dF0", gF), ("dC0", gC),
                                             ("dE", gE), ("dnu", gnu))]
    if sc.n_act:
        pairs.append(("da", das[0], ga))
    errs = assert_grads(pairs, tol=tol, ctx=bounds)
    for s in sims:
        s.close()
    return errs


def _drift_scene(dim):
    if dim == 2:
        return scenes.tiny(2, seed=11, res=128, n_cells=(48, 12), steps=40, v0=(10.0, 0.0), K=2, s=40.0)
    return scenes.tiny(3, seed=12, res=64, n_cells=(24, 8, 8), steps=40, v0=(6.0, 0.0, 0.0), K=2, s=40.0)


@pytest.mark.parametrize("fuse", [0, 1])
@pytest.mark.parametrize("dim,G,halo", [(2, 2, 1), (2, 3, 1), (3, 2, 1), (3, 3, 1), (3, 2, 2)])
def test_slab_drift_across_boundaries_vs_oracle(dim, G, halo, fuse):
    """Particles stream in +x across the slab boundaries (ownership stays with the t = 0
    slab; their stencils move into the neighbour's window): state and every gradient family
    of the whole body vs the oracle, 40 steps with random F0/C0, actuation, floor friction.
    fuse = 1: the fused G2P2G forward, grid t+1's windows summed between two launches."""
    sc = _drift_scene(dim)
    bounds = parallel.slab_partition(sc.x[0], sc.res, sc.dim, G, halo)
    # the scene really crosses: some particle's base_x ends beyond its slab
    traj, w, g = _oracle(sc, 40, 5)
    bx0 = parallel.base_x(sc.x[0], sc.res)
    bxT = np.floor(traj[40][:, 0] * sc.res - 0.5)
    crossed = sum(int(np.sum((bx0 < hi) & (bxT >= hi))) for _, hi in bounds[:-1])
    assert crossed > 0
    _check_slab_run(sc, 40, G, halo, orc=(traj, w, g), fuse=fuse)


@pytest.fixture(scope="module")
def c3_oracle():
    sc = scenes.quadruped_3d(steps=100)
    return sc, _oracle(sc, 100, 9)


@pytest.mark.parametrize("G,fuse", [(2, 0), (3, 0), (2, 1), (3, 1)])
def test_slab_quadruped_c3_vs_oracle(c3_oracle, G, fuse):
    """configs[2] quadruped (29,952 particles, 16 actuators) split into G x-slabs: whole-body
    state and gradients after 100 steps within the north_star's 1e-3 (unfused and fused forward)."""
    sc, orc = c3_oracle
    _check_slab_run(sc, 100, G, orc=orc, fuse=fuse)


def test_slab_single_context_equals_plain():
    """A slab covering the whole domain is the plain path (no windows): equal up to the
    order of P2G's float atomics (last-ulp differences, as between two plain runs)."""
    sc = scenes.tiny(3, seed=13, res=32, n_cells=(6, 6, 6), steps=10)
    a = mpm.MPM(mpm.Config.from_scene(sc, max_steps=10))
    a.set_scene(sc)
    a.forward(10)
    b = mpm.MPM(mpm.Config.from_scene(sc, max_steps=10))
    b.set_slab(0, sc.res, 1)
    b.set_scene(sc)
    mpm.group_forward([b], 10)
    for p, q in zip(a.get_state(10), b.get_state(10)):
        np.testing.assert_allclose(p, q, rtol=1e-6, atol=1e-6 * np.abs(q).max())


def test_slab_escape_is_an_error():
    """A particle that drifts past its slab's halo is an error (MPM_ERR_OUT_OF_SLAB), not a
    silent loss of its neighbour's grid contributions."""
    sc = scenes.tiny(2, seed=14, res=64, n_cells=(16, 16), steps=40, v0=(60.0, 0.0), K=0)
    sims, idxs, bounds = _slab_sims(sc, 40, 2)
    with pytest.raises(mpm.MPMError) as e:
        mpm.group_forward(sims, 40)
    assert e.value.status == "MPM_ERR_OUT_OF_SLAB"


def test_slab_config_errors():
    sc = scenes.tiny(3, seed=15, res=32, n_cells=(6, 6, 6), steps=4)
    cfg = mpm.Config.from_scene(sc, max_steps=4)
    s = mpm.MPM(cfg)
    for lo, hi, h in ((2, 16, 1), (0, 30, 1), (16, 8, 1), (0, 4, 1), (0, 16, 0), (28, 32, 1)):
        with pytest.raises(mpm.MPMError) as e:
            s.set_slab(lo, hi, h)
        assert e.value.status == "MPM_ERR_INVALID_ARG", (lo, hi, h)
    s.set_slab(0, 16, 1)
    # a slab with a neighbour cannot run alone (no communicator, no group)
    sub, idx = parallel.shard_slab(sc, 0, 16)
    t = mpm.MPM(mpm.Config.from_scene(sub, max_steps=4))
    t.set_slab(0, 16, 1)
    t.set_scene(sub)
    with pytest.raises(mpm.MPMError) as e:
        t.forward(1)
    assert e.value.status == "MPM_ERR_CALL_ORDER"
    # set_slab after set_state, and batch > 1
    with pytest.raises(mpm.MPMError) as e:
        t.set_slab(0, 16, 1)
    assert e.value.status in ("MPM_ERR_CALL_ORDER", "MPM_ERR_INVALID_ARG")
    sb = scenes.quadruped_3d(batch=2, steps=4)
    u = mpm.MPM(mpm.Config.from_scene(sb, max_steps=4))
    with pytest.raises(mpm.MPMError) as e:
        u.set_slab(0, 32, 1)
    assert e.value.status == "MPM_ERR_INVALID_ARG"


def test_nccl_transport_single_rank():
    """The NCCL path itself (dlopen of libnccl, ncclCommInitRank, the da all-reduce) on a
    one-rank communicator: a whole-domain slab with a communicator equals the plain run."""
    T = 10
    sc = scenes.tiny(3, seed=16, res=32, n_cells=(6, 6, 6), steps=T, K=2, s=40.0)
    a = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T))
    a.set_scene(sc)
    b = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T))
    b.set_slab(0, sc.res, 1)
    b.comm_init(0, 1, mpm.comm_unique_id())
    b.set_scene(sc)
    w = np.random.default_rng(17).standard_normal((sc.n, 3)).astype(np.float32)  # not the CoM loss (dE = 0)
    for s_ in (a, b):
        s_.forward(T)
        s_.backward(w)
    ga, gb = a.grad(), b.grad()
    for k in ("dx0", "dv0", "dE", "da"):
        assert rel_err(gb[k], ga[k]) < 1e-5, k
