"""GPU parity at BASELINE.json's full sizes.

configs[1] (C2 walker, 2D, 5,824 particles) and configs[2] (C3 quadruped, 3D, 29,952
particles) are compared with the oracle in full.  configs[3] (C4, 1,048,576 particles, the
bench workload and launch configuration) is checked on sampled outputs the oracle computes
one by one -- a particle's next state depends only on particles within 3 cells, so the
oracle steps that neighbourhood alone -- and via properties that hold at any size (mass and
momentum of the grid, bit-exact binning, the exact CoM-gradient closed form)."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm, scenes
from tests.helpers import assert_grads, oracle_cfg, rel_err

pytestmark = pytest.mark.gpu


def _sim(sc, T):
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T))
    sim.set_scene(sc)
    return sim


def _orc_inputs(sc, r=0):
    return (oracle.pack(sc.x[r], sc.v[r], sc.C[r], sc.F[r]),
            [a[r].astype(np.float64) for a in (sc.mass, sc.vol, sc.E, sc.nu)],
            sc.actuator_id[r], sc.act[r].astype(np.float64))


@pytest.mark.parametrize("name,T", [("C2", 500), ("C3", 200)])
def test_full_config_state_and_gradient(name, T):
    """Full C2 (500 steps) / C3 (200 steps) scenes -- the configs' own horizons -- with
    actuation and floor friction: state after T steps within 1e-3,
    gradients of a random linear loss within 1e-3 (north_star), every input family."""
    sc = scenes.CONFIGS[name](steps=T)
    sim = _sim(sc, T)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    cfg = oracle_cfg(sc)
    st, prm, aid, act = _orc_inputs(sc)
    traj = oracle.forward(cfg, st, *prm, aid, act[:T], T)
    ox, ov, oC, oF = oracle.unpack(traj[T], sc.dim)
    for k, a, b in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC)):
        assert rel_err(a, b) < 1e-3, (k, rel_err(a, b))
    rng = np.random.default_rng(7)
    w = rng.standard_normal(traj[T].shape)
    wx, wv, wC, wF = oracle.unpack(w, sc.dim)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    g0, gE, gnu, ga = oracle.backward(cfg, traj, *prm, aid, act[:T], w)
    gx, gv, gC, gF = oracle.unpack(g0, sc.dim)
    assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF),
                  ("dC0", g["dC0"], gC), ("dE", g["dE"], gE), ("dnu", g["dnu"], gnu),
                  ("da", g["da"][0, :T], ga)], ctx=name)


# ---- C4 at full size, bench launch configuration ---------------------------------------------
@pytest.fixture(scope="module")
def c4():
    T = 20
    sc = scenes.slab_3d(steps=T)
    sim = _sim(sc, T)
    sim.forward(T)
    return sc, sim, T


def test_c4_binning_bit_exact(c4):
    sc, sim, T = c4
    for t in (0, T // 2, T - 1):
        x, orig, key, perm, bs = sim.get_binning(t)
        okey, operm, obs = oracle.bin_particles(3, sc.res, x.reshape(1, sc.n, 3))
        np.testing.assert_array_equal(key, okey)
        np.testing.assert_array_equal(perm, operm)
        np.testing.assert_array_equal(bs, obs)


def test_c4_grid_mass_momentum(c4):
    """Sum_i m_i = Sum_p m_p and Sum_i p_i = Sum_p m_p v_p (Eqs. 3, 5) at full size."""
    sc, sim, T = c4
    for t in (0, T - 1):
        m, vbar = sim.get_grid(t)
        x, v, F, Cm = sim.get_state(t)
        mp = sc.mass[0].astype(np.float64)
        assert abs(m.sum(dtype=np.float64) - mp.sum()) < 1e-5 * mp.sum()
        g = np.array(sc.gravity)
        p = (m[0, :, None].astype(np.float64) * (vbar[0].astype(np.float64) - sc.dt * g))
        P = (mp[:, None] * v.astype(np.float64)).sum(0)
        np.testing.assert_allclose(p.sum(0), P, rtol=1e-4, atol=1e-6 * mp.sum())


def _neighbourhood_step(sc, x, v, F, Cm, idx, radius=3):
    """Oracle one step on the particles within `radius` cells (per axis) of particle idx;
    returns the oracle's next state of idx."""
    res = sc.res
    cell = np.floor(x * res - 0.5)
    near = np.all(np.abs(cell - cell[idx]) <= radius, axis=1)
    sub = np.nonzero(near)[0]
    cfg = oracle_cfg(sc)
    st = oracle.pack(x[sub], v[sub], Cm[sub], F[sub])
    prm = [a[0][sub].astype(np.float64) for a in (sc.mass, sc.vol, sc.E, sc.nu)]
    return sub, cfg, st, prm


def test_c4_sampled_particles_one_step(c4):
    """20 sampled particles of the 1M-particle slab: GPU state at t+1 vs the oracle stepping
    each particle's 7^3-cell neighbourhood from the GPU's state at t.  Per particle the
    error is measured against the field's natural scale (reading R16 for sampled outputs:
    x -> domain length 1, v -> max |v|, C -> 4 res max |v|, F -> max |F|): 1e-5 after 1 step."""
    sc, sim, T = c4
    rng = np.random.default_rng(3)
    for t in (0, T - 2):
        x, v, F, Cm = sim.get_state(t)
        x1, v1, F1, C1 = sim.get_state(t + 1)
        act_t = sc.act[0][t:t + 1].astype(np.float64)
        for idx in rng.choice(sc.n, 10, replace=False):
            sub, cfg, st, prm = _neighbourhood_step(sc, x, v, F, Cm, idx)
            traj = oracle.forward(cfg, st, *prm, sc.actuator_id[0][sub], act_t, 1)
            me = int(np.nonzero(sub == idx)[0][0])
            ox, ov, oC, oF = oracle.unpack(traj[1], 3)
            vmax = max(np.abs(v[sub]).max(), np.abs(ov).max())
            for a, b, scale in ((x1[idx], ox[me], 1.0), (v1[idx], ov[me], vmax),
                                (C1[idx], oC[me], 4 * sc.res * vmax), (F1[idx], oF[me], np.abs(oF).max())):
                assert np.abs(a - b).max() < 1e-5 * scale, (t, idx, a, b, scale)


def test_c4_sampled_adjoint_one_step():
    """Adjoint of one step at full size on sampled particles: a seed that is nonzero only
    near a particle gives a gradient at t = 0 that the oracle reproduces from the
    neighbourhood alone (adjoint support is 2 stencils wide)."""
    sc = scenes.slab_3d(steps=1)
    sim = _sim(sc, 1)
    sim.forward(1)
    x, v, F, Cm = sc.x[0], sc.v[0], sc.F[0], sc.C[0]
    rng = np.random.default_rng(4)
    for idx in rng.choice(sc.n, 3, replace=False):
        cell = np.floor(x * sc.res - 0.5)
        seedmask = np.all(np.abs(cell - cell[idx]) <= 1, axis=1)
        S = oracle.S_of(3)
        w = np.zeros((sc.n, S))
        w[seedmask] = rng.standard_normal((seedmask.sum(), S))
        wx, wv, wC, wF = oracle.unpack(w, 3)
        f32 = lambda a: np.ascontiguousarray(a, np.float32)
        sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
        g = sim.grad()
        sub, cfg, st, prm = _neighbourhood_step(sc, x, v, F, Cm, idx, radius=6)
        aid = sc.actuator_id[0][sub]
        act = sc.act[0][:1].astype(np.float64)
        traj = oracle.forward(cfg, st, *prm, aid, act, 1)
        g0, gE, gnu, ga = oracle.backward(cfg, traj, *prm, aid, act, w[sub])
        me = int(np.nonzero(sub == idx)[0][0])
        gx, gv, gC, gF = oracle.unpack(g0, 3)
        assert_grads([("dx0", g["dx0"][idx], gx[me]), ("dv0", g["dv0"][idx], gv[me]),
                      ("dF0", g["dF0"][idx], gF[me]), ("dC0", g["dC0"][idx], gC[me]),
                      ("dE", g["dE"][idx], gE[me])], ctx=int(idx))


def test_c4_com_gradient_closed_form(c4):
    """L = CoM_x(T) at full size (no wall contact in 20 steps): dL/dx0 = m/M e_x, dL/dv0 =
    T dt m/M e_x; dF0, dC0, dE, dnu, da vanish (exactly in real arithmetic)."""
    sc, sim, T = c4
    m = sc.mass[0].astype(np.float64)
    M = m.sum()
    seed = np.zeros((sc.n, 3), np.float32)
    seed[:, 0] = m / M
    sim.backward(seed)
    g = sim.grad()
    ex = np.array([1.0, 0.0, 0.0])
    assert rel_err(g["dx0"], (m / M)[:, None] * ex) < 1e-4
    assert rel_err(g["dv0"], (T * sc.dt * m / M)[:, None] * ex) < 1e-4
    scale = 1.0 / sc.n
    assert np.abs(g["dF0"]).max() < 1e-3 * scale
    assert np.abs(g["dC0"]).max() < 1e-3 * scale * sc.dt
    assert np.abs(g["da"]).max() < 1e-6


def test_batched_quadrupeds_per_rollout():
    """C5b-style batch: 3 quadruped rollouts (own actuation phase and E scale) in one
    context -- the batch dimension folded into the launch grid; each rollout vs the oracle."""
    T = 20
    sc = scenes.quadruped_3d(batch=3, steps=T, e_scale=True)
    sim = _sim(sc, T)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    rng = np.random.default_rng(9)
    S = oracle.S_of(3)
    w = rng.standard_normal((sc.batch, sc.n, S))
    wx, wv, wC, wF = oracle.unpack(w.reshape(-1, S), 3)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    cfg = oracle_cfg(sc)
    for r in range(sc.batch):
        st, prm, aid, act = _orc_inputs(sc, r)
        traj = oracle.forward(cfg, st, *prm, aid, act[:T], T)
        ox, ov, oC, oF = oracle.unpack(traj[T], 3)
        sl = slice(r * sc.n, (r + 1) * sc.n)
        for k, a, b in (("x", x[sl], ox), ("v", v[sl], ov), ("F", F[sl], oF), ("C", Cm[sl], oC)):
            assert rel_err(a, b) < 1e-4, (r, k, rel_err(a, b))
        g0, gE, gnu, ga = oracle.backward(cfg, traj, *prm, aid, act[:T], w[r])
        gx, gv, gC, gF = oracle.unpack(g0, 3)
        assert_grads([("dx0", g["dx0"][sl], gx), ("dv0", g["dv0"][sl], gv), ("dF0", g["dF0"][sl], gF),
                      ("dC0", g["dC0"][sl], gC), ("dE", g["dE"][sl], gE), ("dnu", g["dnu"][sl], gnu),
                      ("da", g["da"][r, :T], ga)], ctx=r)


def test_c5b_full_batch_sampled_rollouts():
    """C5b at full size in bench.py's N = 1 launch configuration: 64 quadruped rollouts
    (1,916,928 particles, per-rollout actuation phase and E scale) in one context, 20 steps
    forward + backward; rollouts 0, 31 and 63 in full vs the oracle (state and gradients)."""
    T = 20
    sc = scenes.quadruped_3d(batch=64, steps=T, e_scale=True)
    sim = _sim(sc, T)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    rng = np.random.default_rng(8)
    S = oracle.S_of(3)
    w = rng.standard_normal((sc.batch * sc.n, S))
    wx, wv, wC, wF = oracle.unpack(w, 3)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    cfg = oracle_cfg(sc)
    for r in (0, 31, 63):
        sl = slice(r * sc.n, (r + 1) * sc.n)
        st, prm, aid, act = _orc_inputs(sc, r)
        traj = oracle.forward(cfg, st, *prm, aid, act[:T], T)
        ox, ov, oC, oF = oracle.unpack(traj[T], 3)
        for k, a, b in (("x", x[sl], ox), ("v", v[sl], ov), ("F", F[sl], oF), ("C", Cm[sl], oC)):
            assert rel_err(a, b) < 1e-4, (r, k, rel_err(a, b))
        g0, gE, gnu, ga = oracle.backward(cfg, traj, *prm, aid, act[:T], w[sl])
        gx, gv, gC, gF = oracle.unpack(g0, 3)
        assert_grads([("dx0", g["dx0"][sl], gx), ("dv0", g["dv0"][sl], gv), ("dF0", g["dF0"][sl], gF),
                      ("dC0", g["dC0"][sl], gC), ("dE", g["dE"][sl], gE), ("dnu", g["dnu"][sl], gnu),
                      ("da", g["da"][r, :T], ga)], ctx=r)


def test_c4_fused_sampled_neighbourhoods_multi_step():
    """The exact bench path at C4 (fused G2P2G forward, whole-block backward, 1,048,576
    particles) over T = 6 steps, against the oracle on sampled neighbourhoods: a random seed on
    every state family of the particles within one cell of a sampled particle; the oracle
    runs forward + backward on the particles within R = 2T + 2 cells of it (the dependency cone
    of T steps: a particle's base cell reaches +-2 cells per step; measured with the oracle
    itself on a 166k-particle slab, the truncation error is exactly 0 at R = 2T + 2).  Compared
    element-wise: state at T and dL/dx0, dv0, dF0, dC0, dE, dnu of the seeded particles, and the
    whole dL/da[t][k] (every actuator sum only sees particles inside the cone)."""
    from tests.helpers import assert_grads
    T = 6
    sc = scenes.slab_3d(steps=T)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, fuse_g2p2g=1))
    sim.set_scene(sc)
    sim.forward(T)
    xT, vT, FT, CT = sim.get_state(T)
    x0 = sc.x[0]
    cell = np.floor(x0 * sc.res - 0.5)
    lo, hi = cell.min(0), cell.max(0)
    rng = np.random.default_rng(12)
    S = oracle.S_of(3)
    cfg = oracle_cfg(sc)
    act = sc.act[0][:T].astype(np.float64)
    picks = [  # interior, a top corner of the slab (free surface), a bottom edge
        np.argmin(np.abs(cell - (lo + hi) / 2).sum(1)),
        np.argmin(np.abs(cell - np.array([lo[0], hi[1], hi[2]])).sum(1)),
        np.argmin(np.abs(cell - np.array([(lo[0] + hi[0]) / 2, lo[1], lo[2] + 3])).sum(1)),
    ]
    R = 2 * T + 2
    for idx in picks:
        seedmask = np.all(np.abs(cell - cell[idx]) <= 1, axis=1)
        w = np.zeros((sc.n, S))
        w[seedmask] = rng.standard_normal((seedmask.sum(), S))
        wx, wv, wC, wF = oracle.unpack(w, 3)
        f32 = lambda a: np.ascontiguousarray(a, np.float32)
        sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
        g = sim.grad()
        sub = np.nonzero(np.all(np.abs(cell - cell[idx]) <= R, axis=1))[0]
        st = oracle.pack(sc.x[0][sub], sc.v[0][sub], sc.C[0][sub], sc.F[0][sub])
        prm = [a[0][sub].astype(np.float64) for a in (sc.mass, sc.vol, sc.E, sc.nu)]
        aid = sc.actuator_id[0][sub]
        traj = oracle.forward(cfg, st, *prm, aid, act, T)
        g0, gE, gnu, ga = oracle.backward(cfg, traj, *prm, aid, act, w[sub])
        cmp = np.nonzero(seedmask)[0]
        pos = np.searchsorted(sub, cmp)
        ox, ov, oC, oF = oracle.unpack(traj[T][pos], 3)
        vmax = np.abs(oracle.unpack(traj[T], 3)[1]).max()
        for k, a, b, scale in (("x", xT[cmp], ox, 1.0), ("v", vT[cmp], ov, vmax), ("F", FT[cmp], oF, np.abs(oF).max()),
                               ("C", CT[cmp], oC, 4 * sc.res * vmax)):
            assert np.abs(a - b).max() / scale < 1e-4, (idx, k)
        gx, gv, gC, gF = oracle.unpack(g0[pos], 3)
        assert_grads([("dx0", g["dx0"][cmp], gx), ("dv0", g["dv0"][cmp], gv), ("dF0", g["dF0"][cmp], gF),
                      ("dC0", g["dC0"][cmp], gC), ("dE", g["dE"][cmp], gE[pos]), ("dnu", g["dnu"][cmp], gnu[pos]),
                      ("da", g["da"][0, :T], ga)], ctx=int(idx))
