"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the same
seeded fp32 inputs.  Bars (BASELINE.json north_star): binning bit-exact; state within 1e-5
relative after 1 step and 1e-3 after 100 steps; gradients within 1e-3 relative
(norm-wise per field, reading R16)."""
import os

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


def _oracle_traj(sc, r, T):
    cfg = oracle_cfg(sc)
    m, vol, E, nu, aid, act = oracle_params(sc, r)
    return cfg, oracle.forward(cfg, oracle_state(sc, r), m, vol, E, nu, aid, act[:T], T)


def _split(sc, arr, r):
    return arr.reshape(sc.batch, sc.n, *arr.shape[1:])[r]


# ---- binning: bit-exact ---------------------------------------------------------------
@pytest.mark.parametrize("name,kw,T", [
    ("tiny2", dict(dim=2, seed=1, res=32, n_cells=(9, 7), steps=6), 6),
    ("tiny3", dict(dim=3, seed=2, res=16, n_cells=(5, 4, 6), steps=6), 6),
    ("dense3", dict(dim=3, seed=3, res=32, n_cells=(12, 8, 9), steps=4), 4),
])
def test_binning_bit_exact(name, kw, T):
    sc = scenes.tiny(**kw)
    sim = _sim(sc, T)
    sim.forward(T)
    for t in range(T):
        x, orig, key, perm, bs = sim.get_binning(t)
        okey, operm, obs = oracle.bin_particles(sc.dim, sc.res, x.reshape(sc.batch, sc.n, sc.dim))
        np.testing.assert_array_equal(key, okey)
        np.testing.assert_array_equal(perm, operm)
        np.testing.assert_array_equal(bs, obs)
        assert sorted(orig.tolist()) == list(range(sc.batch * sc.n))


def test_binning_batch_and_oversize_block():
    """Several rollouts, one block holding > 2048 particles (in-smem sort capacity) and
    particles piled into single cells (ties)."""
    rng = np.random.default_rng(5)
    sc = scenes.tiny(3, seed=5, res=32, n_cells=(4, 4, 4), steps=2, K=0)
    n = 3000
    d = 3
    x = np.empty((2, n, d), np.float32)
    x[:, :, :] = (rng.uniform(16.6, 19.4, (2, n, d)) / 32).astype(np.float32)  # one 4^3 block
    x[:, :500] = x[:, :1]
    v = (0.1 * rng.standard_normal((2, n, d))).astype(np.float32)
    cfg = mpm.Config(dim=3, res=32, batch=2, n_particles=n, max_steps=2, dt=1e-5)
    sim = mpm.MPM(cfg)
    NT = 2 * n
    one = np.ones(NT, np.float32)
    sim.set_state(x.reshape(NT, d), v.reshape(NT, d), None, None, one * 1e-6, one * 1e-6,
                  one * 1e3, one * 0.3, None)
    sim.forward(2)
    for t in range(2):
        xs, orig, key, perm, bs = sim.get_binning(t)
        okey, operm, obs = oracle.bin_particles(3, 32, xs.reshape(2, n, 3))
        np.testing.assert_array_equal(key, okey)
        np.testing.assert_array_equal(perm, operm)
        np.testing.assert_array_equal(bs, obs)


# ---- grid of one step -------------------------------------------------------------------
@pytest.mark.parametrize("d", [2, 3])
def test_grid_parity_step0(d):
    sc = scenes.tiny(d, seed=7, res=16, steps=1, K=2, s=50.0)
    sim = _sim(sc, 1)
    sim.forward(1)
    m, vbar = sim.get_grid(0)
    cfg = oracle_cfg(sc)
    mp, vol, E, nu, aid, act = oracle_params(sc)
    om, op, ovbar, ov = oracle.step_grid(cfg, oracle_state(sc), mp, vol, E, nu, aid, act[0])
    assert rel_err(m[0], om) < 1e-6
    assert rel_err(vbar[0], ovbar) < 1e-5


# ---- forward state ------------------------------------------------------------------------
@pytest.mark.parametrize("d,T,tol", [(2, 1, 1e-5), (3, 1, 1e-5), (2, 100, 1e-3), (3, 100, 1e-3)])
def test_forward_state_parity(d, T, tol):
    sc = scenes.tiny(d, seed=11 + d, res=16 if d == 3 else 32, n_cells=(4,) * d, steps=T, K=2,
                     s=40.0, center=(6,) * d if d == 3 else (12, 4))
    sim = _sim(sc, T)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    _, traj = _oracle_traj(sc, 0, T)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    for name, a, b in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC)):
        e = rel_err(a, b)
        assert e < tol, (name, e)


def test_forward_c1_full_50_steps():
    """configs[0] (C1) at its full size: 1,024 particles, 50 steps, every rollout."""
    sc = scenes.block_2d(steps=50, perturb=True, batch=2)
    sim = _sim(sc, 50)
    sim.forward(50)
    x, v, F, Cm = sim.get_state(50)
    for r in range(2):
        _, traj = _oracle_traj(sc, r, 50)
        ox, ov, oC, oF = oracle.unpack(traj[50], 2)
        for name, a, b in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC)):
            assert rel_err(_split(sc, a, r), b) < 1e-3, (r, name)


# ---- gradients -------------------------------------------------------------------------------
def _grad_case(sc, T, seed=0):
    sim = _sim(sc, T)
    sim.forward(T)
    cfg, traj = _oracle_traj(sc, 0, T)
    rng = np.random.default_rng(seed)
    w = rng.standard_normal(traj[T].shape)
    wx, wv, wC, wF = oracle.unpack(w, sc.dim)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    m, vol, E, nu, aid, act = oracle_params(sc)
    g0, gE, gnu, ga = oracle.backward(cfg, traj, m, vol, E, nu, aid, act[:T], w)
    gx, gv, gC, gF = oracle.unpack(g0, sc.dim)
    return g, dict(dx0=gx, dv0=gv, dF0=gF, dC0=gC, dE=gE, dnu=gnu, da=ga)


@pytest.mark.parametrize("d,T", [(2, 10), (3, 10), (3, 40)])
def test_gradient_parity(d, T):
    sc = scenes.tiny(d, seed=21 + d, res=16 if d == 3 else 32, n_cells=(4,) * d, steps=T, K=2,
                     s=40.0, center=(6, 4, 6) if d == 3 else (12, 4))
    g, o = _grad_case(sc, T)
    assert_grads([(k, g[k], o[k]) for k in ("dx0", "dv0", "dF0", "dC0", "dE", "dnu")] +
                 [("da", g["da"][0, :T], o["da"])])


def test_com_gradient_closed_form_gpu():
    """L = CoM_x(T) without wall contact: dL/dx0 = m/M e_x, dL/dv0 = T dt m/M e_x exactly."""
    T = 30
    sc = scenes.tiny(3, seed=31, res=16, K=2, s=40.0, steps=T, center=(6, 6, 6))
    sc.v[:] *= 0.05
    sim = _sim(sc, T)
    sim.forward(T)
    m = sc.mass[0].astype(np.float64)
    seed = np.zeros((sc.n, 3), np.float32)
    seed[:, 0] = m / m.sum()
    sim.backward(seed)
    g = sim.grad()
    ex = np.zeros(3)
    ex[0] = 1
    assert rel_err(g["dx0"], (m / m.sum())[:, None] * ex) < 1e-4
    assert rel_err(g["dv0"], (T * sc.dt * m / m.sum())[:, None] * ex) < 1e-4
    scale = 1.0 / sc.n
    assert np.abs(g["dF0"]).max() < 1e-4 * scale * T
    assert np.abs(g["da"]).max() < 1e-6


# ---- error paths ------------------------------------------------------------------------------
def test_errors_out_of_domain_and_inverted_and_call_order():
    sc = scenes.tiny(3, seed=41, res=16, K=0, steps=2)
    cfg = mpm.Config.from_scene(sc, max_steps=2)
    sim = mpm.MPM(cfg)
    with pytest.raises(mpm.MPMError) as e:
        sim.forward(1)
    assert e.value.status == "MPM_ERR_CALL_ORDER"
    x = sc.x[0].copy()
    x[3, 1] = 0.01
    with pytest.raises(mpm.MPMError) as e:
        sim.set_state(x, sc.v[0], sc.F[0], sc.C[0], sc.mass[0], sc.vol[0], sc.E[0], sc.nu[0])
    assert e.value.status == "MPM_ERR_OUT_OF_DOMAIN"
    F = sc.F[0].copy()
    F[5] = np.diag([-1.0, 1.0, 1.0])
    sim.set_state(sc.x[0], sc.v[0], F, sc.C[0], sc.mass[0], sc.vol[0], sc.E[0], sc.nu[0])
    with pytest.raises(mpm.MPMError) as e:
        sim.forward(1)
    assert e.value.status == "MPM_ERR_INVERTED"
    with pytest.raises(mpm.MPMError) as e:
        sim.forward(1)
    assert e.value.status == "MPM_ERR_CALL_ORDER"
    sim.set_state(sc.x[0], sc.v[0], sc.F[0], sc.C[0], sc.mass[0], sc.vol[0], sc.E[0], sc.nu[0])
    sim.forward(2)
    with pytest.raises(mpm.MPMError) as e:
        sim.forward(1)
    assert e.value.status == "MPM_ERR_TAPE_FULL"


@pytest.mark.parametrize("d,T", [(2, 10), (3, 12)])
def test_mass_gradient_and_running_loss_parity(d, T):
    """NEXT N3 (dL/dm_p) and N4 (seeds at intermediate states: a running loss
    sum_t <w_t, state_t>) against the oracle's orc_backward_ex."""
    sc = scenes.tiny(d, seed=51 + d, res=16 if d == 3 else 32, n_cells=(4,) * d, steps=T, K=2,
                     s=40.0, center=(6, 4, 6) if d == 3 else (12, 4))
    sim = _sim(sc, T)
    sim.enable_mass_grad(True)
    sim.forward(T)
    cfg, traj = _oracle_traj(sc, 0, T)
    rng = np.random.default_rng(52 + d)
    W = rng.standard_normal(traj.shape)
    W[1::2] = 0.0  # seeds on every other state (and always on the last)
    W[T] = rng.standard_normal(traj[T].shape)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    for t in range(T):
        if np.any(W[t]):
            wx, wv, wC, wF = oracle.unpack(W[t], d)
            sim.add_seed(t, f32(wx), f32(wv), f32(wF), f32(wC))
    wx, wv, wC, wF = oracle.unpack(W[T], d)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    gm = sim.grad_mass()
    m, vol, E, nu, aid, act = oracle_params(sc)
    g0, gE, gnu, ga, ogm = oracle.backward_ex(cfg, traj, m, vol, E, nu, aid, act[:T], W)
    gx, gv, gC, gF = oracle.unpack(g0, d)
    assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF),
                  ("dC0", g["dC0"], gC), ("dE", g["dE"], gE), ("dm", gm, ogm)])
    sim.clear_seeds()
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g2 = sim.grad()
    g0b, *_ = oracle.backward(cfg, traj, m, vol, E, nu, aid, act[:T], W[T])
    assert_grads([("dx0", g2["dx0"], oracle.unpack(g0b, d)[0])])


def test_c_abi_demo_program(tmp_path):
    """The boundary is a plain C ABI: examples/c_api_demo.c (no Python, no torch) builds
    with gcc against include/mpm.h + libmpm.so and reproduces the CoM closed form."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "c_api_demo")
    lib = os.path.join(root, "paper_1810_01054_b200")
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", "c_api_demo.c"), "-L", lib, "-lmpm",
                           f"-Wl,-rpath,{lib}", "-lm", "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
