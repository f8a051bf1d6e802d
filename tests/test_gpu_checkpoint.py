"""NEXT N2 on the GPU: long-horizon memory by checkpoint + segment recompute
(config.checkpoint_every = k).  The checkpointed run must give the memo run's state and
gradients (up to the order of P2G's float atomics in the recomputed forward) and the oracle's;
the 1000-step free-flight case is the paper's long-horizon check at C4 size."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm, scenes
from tests.helpers import assert_grads, oracle_cfg, oracle_params, oracle_state, rel_err

pytestmark = pytest.mark.gpu


def _sim(sc, T, k, **kw):
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, checkpoint_every=k, **kw))
    sim.set_scene(sc)
    return sim


def _seed(sc, seed=3):
    S = oracle.S_of(sc.dim)
    w = np.random.default_rng(seed).standard_normal((sc.batch * sc.n, S))
    wx, wv, wC, wF = oracle.unpack(w, sc.dim)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    return w, (f32(wx), f32(wv), f32(wF), f32(wC))


@pytest.mark.parametrize("k", [1, 7, 30])
def test_checkpointed_equals_memo_and_oracle(k):
    T = 30
    sc = scenes.tiny(3, seed=51, res=32, n_cells=(6, 6, 6), steps=T, K=2, s=40.0)
    w, seeds = _seed(sc)
    a = _sim(sc, T, 0)
    b = _sim(sc, T, k)
    a.forward(T)
    b.forward(T)
    for p, q in zip(a.get_state(T), b.get_state(T)):
        assert rel_err(q, p) < 1e-6
    a.backward(*seeds)
    b.backward(*seeds)
    ga, gb = a.grad(), b.grad()
    for key in ("dx0", "dv0", "dF0", "dC0", "dE", "dnu", "da"):
        assert rel_err(gb[key], ga[key]) < 1e-4, (key, rel_err(gb[key], ga[key]))
    cfg = oracle_cfg(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    g0, gE, gnu, gact = oracle.backward(cfg, traj, m, vol, E, nu, aid, act[:T], w)
    gx, gv, gC, gF = oracle.unpack(g0, 3)
    assert_grads([(key, gb[key], ref) for key, ref in (("dx0", gx), ("dv0", gv), ("dF0", gF), ("dC0", gC),
                                                       ("dE", gE), ("dnu", gnu))] + [("da", gb["da"][0, :T], gact)])


def test_checkpointed_with_controller_seeds_and_mass_grad():
    """N1 controller, N4 running-loss seeds at several steps (inside and at segment
    boundaries) and the N3 mass gradient all survive the segment recompute."""
    T, k = 24, 5
    sc = scenes.tiny(2, seed=52, res=32, n_cells=(8, 8), steps=T, K=3, s=40.0)
    K, d = sc.n_act, 2
    nz = d * (1 + 2 * K)
    rng = np.random.default_rng(8)
    W = (rng.standard_normal((K * d, nz)) * 0.3).astype(np.float32)
    bb = rng.uniform(-0.5, 0.5, K * d).astype(np.float32)
    target = np.array([0.6, 0.4], np.float32)
    out = []
    for kk in (0, k):
        s = _sim(sc, T, kk)
        s.set_controller(W, bb, target)
        s.enable_mass_grad(True)
        for t in (0, 5, 12, 20):
            _, sd = _seed(sc, 100 + t)
            s.add_seed(t, *sd)
        s.forward(T)
        s.backward(*_seed(sc)[1])
        out.append((s.grad(), s.grad_controller(), s.grad_mass()))
    (g0, c0, m0), (g1, c1, m1) = out
    for key in ("dx0", "dv0", "dF0", "dC0", "dE", "dnu", "da"):
        assert rel_err(g1[key], g0[key]) < 1e-4, key
    for x, y in zip(c1, c0):
        assert rel_err(x, y) < 1e-4
    assert rel_err(m1, m0) < 1e-4


def test_evicted_state_is_recomputed_and_rewind_works():
    T, k = 20, 6
    sc = scenes.tiny(3, seed=53, res=32, n_cells=(5, 5, 5), steps=T, K=2, s=40.0)
    a = _sim(sc, T, 0)
    b = _sim(sc, T, k)
    a.forward(T)
    b.forward(T)
    for t in (3, 6, 11, 20):  # 3 and 11 are evicted: recomputed from checkpoints 0 and 1
        for p, q in zip(a.get_state(t), b.get_state(t)):
            assert rel_err(q, p) < 1e-6, t
    # introspection needs residency (step 4's tables: states 4 and 5 on the tape)
    b.get_state(5)
    b.step_info(4)
    with pytest.raises(mpm.MPMError):
        b.step_info(15)
    # rewind into an evicted segment, then run on with a changed actuation
    b.rewind(9)
    a.rewind(9)
    act = np.zeros((1, T, sc.n_act, 3), np.float32)
    act[:, :, :, 1] = 0.5
    a.set_actuation(act)
    b.set_actuation(act)
    a.forward(T - 9)
    b.forward(T - 9)
    for p, q in zip(a.get_state(T), b.get_state(T)):
        assert rel_err(q, p) < 1e-6
    # a second backward after the first evicted the tape end
    _, seeds = _seed(sc)
    b.backward(*seeds)
    g1 = b.grad()["dx0"].copy()
    b.backward(*seeds)
    assert rel_err(b.grad()["dx0"], g1) < 1e-5


def test_long_horizon_1000_steps_c4_free_flight():
    """1000 steps of free flight; with no wall contact and g = 0 the CoM moves
    exactly with the initial momentum for any internal stress and actuation, so for
    L = CoM_x(T): dL/dx0_p = m_p/M e_x, dL/dv0_p = T dt m_p/M e_x.  C4 size (1,048,576
    particles): the memo would need ~100 GB; checkpoint_every = 50 needs ~7 GB."""
    T, k = 1000, 50
    sc = scenes.slab_3d(steps=T, y0=20)
    sc.gravity = (0.0, 0.0, 0.0)
    sc.v[..., 0] = 0.3
    sc.v[..., 1] = 0.0
    sim = _sim(sc, T, k)
    sim.forward(T)
    m = sc.mass[0].astype(np.float64)
    M = m.sum()
    seed = np.zeros((sc.n, 3), np.float32)
    seed[:, 0] = (m / M).astype(np.float32)
    x = sim.get_state(T)[0].astype(np.float64)
    com0 = (m[:, None] * sc.x[0]).sum(0) / M
    comT = (m[:, None] * x).sum(0) / M
    np.testing.assert_allclose(comT - com0, [0.3 * T * sc.dt, 0.0, 0.0], atol=1e-5)
    sim.backward(seed)
    g = sim.grad()
    ex = np.zeros(3)
    ex[0] = 1.0
    assert rel_err(g["dx0"], (m / M)[:, None] * ex) < 1e-3
    assert rel_err(g["dv0"], (T * sc.dt * m / M)[:, None] * ex) < 1e-3
    # the remaining families vanish (relative to the x0 gradient's per-particle scale)
    scale = np.abs(g["dx0"]).max()
    assert np.abs(g["dF0"]).max() < 1e-2 * scale and np.abs(g["dC0"]).max() < 1e-2 * scale * sc.dt * 100
