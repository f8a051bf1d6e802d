"""NEXT N2 fused forward (config.fuse_g2p2g = 1: one particle pass per step, k_g2p2g) against
the fp64 oracle and against the unfused path: the same bars as the unfused parity tests
(state 1e-5 after 1 step / 1e-3 after 100 steps, gradients 1e-3, binning bit-exact), the
memo grid equal up to fp32 summation order, checkpoint recompute and forward calls split
into pieces, the full C4 slab, and the CFL error when a particle outruns the dilation."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm, scenes
from tests.helpers import assert_grads, oracle_cfg, oracle_params, oracle_state, rel_err

pytestmark = pytest.mark.gpu


def _sim(sc, T, **kw):
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, **kw))
    sim.set_scene(sc)
    return sim


def _tiny(d, T, seed):
    return scenes.tiny(d, seed=seed + d, res=16 if d == 3 else 32, n_cells=(4,) * d, steps=T, K=2,
                       s=40.0, center=(6,) * d if d == 3 else (12, 4))


@pytest.mark.parametrize("d,T,tol", [(2, 1, 1e-5), (3, 1, 1e-5), (2, 100, 1e-3), (3, 100, 1e-3)])
def test_fused_forward_state_parity(d, T, tol):
    sc = _tiny(d, T, 11)
    sim = _sim(sc, T, fuse_g2p2g=1)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    cfg = oracle_cfg(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    for name, a, b in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC)):
        assert rel_err(a, b) < tol, (name, rel_err(a, b))


@pytest.mark.parametrize("d,T", [(2, 10), (3, 10), (3, 40)])
def test_fused_gradient_parity(d, T):
    sc = _tiny(d, T, 21)
    sim = _sim(sc, T, fuse_g2p2g=1)
    sim.forward(T)
    cfg = oracle_cfg(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    w = np.random.default_rng(0).standard_normal(traj[T].shape)
    wx, wv, wC, wF = oracle.unpack(w, d)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    g0, gE, gnu, ga = oracle.backward(cfg, traj, m, vol, E, nu, aid, act[:T], w)
    gx, gv, gC, gF = oracle.unpack(g0, d)
    assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF),
                  ("dC0", g["dC0"], gC), ("dE", g["dE"], gE), ("dnu", g["dnu"], gnu),
                  ("da", g["da"][0, :T], ga)])


@pytest.mark.parametrize("name,make,T", [
    ("C1 2D block, 50 steps", lambda: scenes.block_2d(steps=50, perturb=True, batch=2), 50),
    ("C2 2D walker, 100 steps", lambda: scenes.walker_2d(steps=100), 100),
    ("C3 3D quadruped, 60 steps", lambda: scenes.quadruped_3d(steps=60), 60),
])
def test_fused_baseline_configs_vs_oracle(name, make, T):
    """The small BASELINE configs through the fused forward (particles cross block faces in
    every direction, 2D blocks are 8 cells wide): state vs the oracle (1e-3), every rollout."""
    sc = make()
    sim = _sim(sc, T, fuse_g2p2g=1)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    for r in range(sc.batch):
        cfg = oracle_cfg(sc)
        m, vol, E, nu, aid, act = oracle_params(sc, r)
        traj = oracle.forward(cfg, oracle_state(sc, r), m, vol, E, nu, aid, act[:T], T)
        ox, ov, oC, oF = oracle.unpack(traj[T], sc.dim)
        sl = slice(r * sc.n, (r + 1) * sc.n)
        for k, a, b in (("x", x[sl], ox), ("v", v[sl], ov), ("F", F[sl], oF), ("C", Cm[sl], oC)):
            assert rel_err(a, b) < 1e-3, (name, r, k, rel_err(a, b))


def test_fused_binning_bit_exact_and_grid_equal():
    """The fused run's binning (its own in-kernel cell sort) is bit-exact with the oracle's,
    and its memo grid (dilated slot map) holds the unfused (p, m) up to summation order."""
    T = 6
    sc = scenes.tiny(3, seed=3, res=32, n_cells=(12, 8, 9), steps=T)
    fu = _sim(sc, T, fuse_g2p2g=1)
    ref = _sim(sc, T)
    fu.forward(T)
    ref.forward(T)
    for t in range(T):
        x, orig, key, perm, bs = fu.get_binning(t)
        okey, operm, obs = oracle.bin_particles(3, sc.res, x.reshape(1, sc.n, 3))
        np.testing.assert_array_equal(key, okey)
        np.testing.assert_array_equal(perm, operm)
        np.testing.assert_array_equal(bs, obs)
        (mf, vf), (mr, vr) = fu.get_grid(t), ref.get_grid(t)
        np.testing.assert_allclose(mf, mr, rtol=1e-5, atol=1e-6 * mr.max())
        touched = mr > 0
        assert np.all((mf > 0) == touched)
        assert rel_err(vf[touched], vr[touched]) < 1e-5
    info_f = [fu.step_info(t) for t in range(T)]
    info_r = [ref.step_info(t) for t in range(T)]
    assert info_f[0] == info_r[0]  # step 0: the unfused P2G builds the grid
    assert all(f[1] >= r[1] for f, r in zip(info_f[1:], info_r[1:]))  # dilated slot maps


def test_fused_matches_unfused_c4_slab():
    """configs[3] (C4: 1,048,576 particles) at full size, 20 steps: the fused and unfused
    paths agree on the state (1e-5) and on the CoM gradient (closed form, 1e-4)."""
    T = 20
    sc = scenes.slab_3d(steps=T)
    out = []
    for fuse in (0, 1):
        sim = _sim(sc, T, fuse_g2p2g=fuse)
        sim.forward(T)
        x, v, F, Cm = sim.get_state(T)
        m = sc.mass[0].astype(np.float64)
        seed = np.zeros((sc.n, 3), np.float32)
        seed[:, 0] = m / m.sum()
        sim.backward(seed)
        out.append((x, v, F, Cm, sim.grad()))
        sim.close()
    (x0, v0, F0, C0, g0), (x1, v1, F1, C1, g1) = out
    assert rel_err(x1, x0) < 1e-6
    assert rel_err(v1, v0) < 1e-4 and rel_err(F1, F0) < 1e-5 and rel_err(C1, C0) < 1e-4
    m = sc.mass[0].astype(np.float64)
    ex = np.array([1.0, 0.0, 0.0])
    assert rel_err(g1["dx0"], (m / m.sum())[:, None] * ex) < 1e-4
    assert rel_err(g1["dv0"], (T * sc.dt * m / m.sum())[:, None] * ex) < 1e-4


@pytest.mark.parametrize("k", [1, 7])
def test_fused_checkpoint_and_split_calls(k):
    """Checkpoint segments (the backward recomputes them through the fused path) and a
    forward split into several calls give the single-call unfused result."""
    T = 30
    sc = _tiny(3, T, 31)
    ref = _sim(sc, T)
    ref.forward(T)
    fu = _sim(sc, T, fuse_g2p2g=1, checkpoint_every=k)
    for n in (4, 1, 11, 14):
        fu.forward(n)
    for a, b in zip(fu.get_state(T), ref.get_state(T)):
        assert rel_err(a, b) < 1e-5
    rng = np.random.default_rng(3)
    seeds = [rng.standard_normal((sc.n, 3)).astype(np.float32) for _ in range(2)]
    ref.backward(*seeds)
    fu.backward(*seeds)
    gr, gf = ref.grad(), fu.grad()
    for key in ("dx0", "dv0", "dF0", "dC0", "dE", "dnu", "da"):
        assert rel_err(gf[key], gr[key]) < 1e-4, key


def test_fused_fixed_corotated():
    T = 20
    sc = _tiny(3, T, 41)
    ref = _sim(sc, T, material=1)
    fu = _sim(sc, T, material=1, fuse_g2p2g=1)
    ref.forward(T)
    fu.forward(T)
    for a, b in zip(fu.get_state(T), ref.get_state(T)):
        assert rel_err(a, b) < 1e-5


def test_fused_launches_one_particle_pass_per_step():
    T = 12
    sc = _tiny(3, T, 51)
    sim = _sim(sc, T, fuse_g2p2g=1)
    sim.set_profiling(True)
    sim.forward(T)
    prof = sim.profile()
    assert prof["p2g"][1] == 1          # only the first step's grid is built unfused
    assert prof["g2p2g"][1] == T        # every step: one fused particle pass
    assert prof["g2p"][1] == 0


def test_fused_cfl_violation_is_an_error():
    """A lone particle moving 3 cells in one step leaves the dilated grid: MPM_ERR_CFL."""
    res, dt = 32, 1e-3
    sc = scenes.tiny(3, seed=61, res=res, steps=3, K=0)
    n = 1
    sc.x = np.array([[[(4 * 3 + 3.6) / res, 0.5, 0.5]]], np.float32)
    sc.v = np.array([[[3.0 / (res * dt), 0.0, 0.0]]], np.float32)
    sc.F = np.eye(3, dtype=np.float32)[None, None]
    sc.C = np.zeros((1, n, 3, 3), np.float32)
    for f in ("mass", "vol"):
        setattr(sc, f, np.full((1, n), 1e-6, np.float32))
    sc.E = np.full((1, n), 1e3, np.float32)
    sc.nu = np.full((1, n), 0.3, np.float32)
    sc.actuator_id = np.full((1, n), -1, np.int32)
    sc.gravity = (0.0, 0.0, 0.0)
    sc.dt = dt
    sim = _sim(sc, 3, fuse_g2p2g=1)
    with pytest.raises(mpm.MPMError) as e:
        sim.forward(3)
    assert e.value.status == "MPM_ERR_CFL"


def test_fused_mass_gradient_and_running_seeds_match_unfused():
    """The backward features that read the memo grid (N3 dL/dm_p, N4 seeds at intermediate
    states) give the unfused results over the fused forward's dilated grids."""
    T = 16
    sc = _tiny(3, T, 61)
    rng = np.random.default_rng(8)
    seeds = {t: [rng.standard_normal((sc.n, 3)).astype(np.float32) for _ in range(2)] for t in (5, 11)}
    fin = [rng.standard_normal((sc.n, 3)).astype(np.float32) for _ in range(2)]
    out = []
    for fuse in (0, 1):
        sim = _sim(sc, T, fuse_g2p2g=fuse)
        sim.enable_mass_grad(True)
        for t, (sx, sv) in seeds.items():
            sim.add_seed(t, sx, sv)
        sim.forward(T)
        sim.backward(*fin)
        out.append((sim.grad(), sim.grad_mass()))
        sim.close()
    (g0, m0), (g1, m1) = out
    for key in ("dx0", "dv0", "dF0", "dC0", "dE", "dnu", "da"):
        assert rel_err(g1[key], g0[key]) < 1e-4, key
    assert rel_err(m1, m0) < 1e-4


def test_fused_flag_ignored_with_controller():
    """N1 needs state t+1 before step t+1's P2G: with a controller the fused flag runs the
    unfused forward (same results, no g2p2g launches)."""
    from oracle import controller as ctl
    T = 8
    sc = _tiny(3, T, 71)
    K, d = sc.n_act, 3
    rng = np.random.default_rng(9)
    W = (0.1 * rng.standard_normal((K * d, ctl.n_obs(d, K)))).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, K * d).astype(np.float32)
    target = rng.uniform(0.2, 0.8, d).astype(np.float32)
    res = []
    for fuse in (0, 1):
        sim = _sim(sc, T, fuse_g2p2g=fuse)
        sim.set_controller(W, b, target)
        sim.set_profiling(True)
        sim.forward(T)
        assert sim.profile()["g2p2g"][1] == 0
        res.append(sim.get_state(T))
        sim.close()
    for a, b in zip(*res):
        assert rel_err(a, b) < 1e-6


@pytest.mark.parametrize("d", [2, 3])
def test_fused_fast_diagonal_motion_escapees(d):
    """A body moving 0.9 cells per step along the diagonal: every step a large share of the
    particles leaves its block (escapees of the fused scatter) in every axis direction.  Both
    forwards against the oracle at field scale (R16: C against 4 res |v|, whose fp32
    cancellation under a large common-mode velocity depends on the summation order), and both
    gradients against the oracle's."""
    T = 10
    res = 32
    sc = scenes.tiny(d, seed=81 + d, res=res, n_cells=(6,) * d, steps=T, K=0,
                     center=(10,) * d)
    sc.gravity = (0.0,) * d
    sign = np.array([1.0, -1.0, 1.0][:d])
    sc.v[...] = (0.9 / (res * sc.dt) * sign / np.sqrt(d)).astype(np.float32)
    cfg = oracle_cfg(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    w = np.random.default_rng(4).standard_normal(traj[T].shape)
    wx, wv, wC, wF = oracle.unpack(w, d)
    g0, gE, gnu, _ = oracle.backward(cfg, traj, m, vol, E, nu, aid, act[:T], w)
    gx, gv, gC, gF = oracle.unpack(g0, d)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    bb = 4 if d == 3 else 8
    for fuse in (0, 1):
        sim = _sim(sc, T, fuse_g2p2g=fuse)
        sim.forward(T)
        x, v, F, Cm = sim.get_state(T)
        if fuse:
            moved = np.any(np.floor(x * res - 0.5) // bb != np.floor(sc.x[0] * res - 0.5) // bb, axis=1)
            assert moved.mean() > 0.5  # the escapee path is exercised
        vmax = np.abs(ov).max()
        for k, a, b, scale in (("x", x, ox, 1.0), ("v", v, ov, vmax), ("F", F, oF, np.abs(oF).max()),
                               ("C", Cm, oC, 4 * res * vmax)):
            assert np.abs(a - b).max() / scale < 1e-5, (fuse, k, np.abs(a - b).max() / scale)
        sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
        g = sim.grad()
        assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF),
                      ("dC0", g["dC0"], gC), ("dE", g["dE"], gE), ("dnu", g["dnu"], gnu)], ctx=fuse)
        sim.close()
