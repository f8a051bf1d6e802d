"""NEXT N3 on the GPU: the fixed-corotated material (config.material = 1, DESIGN R21) --
state and every gradient family vs the oracle, whose fixed-corotated path follows the paper's
dP/dF route (dR/dF of the polar decomposition) while the kernels use the Kirchhoff form with a
Lyapunov solve on the left stretch: independent derivations."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm, scenes
from tests.helpers import assert_grads, oracle_cfg, oracle_params, oracle_state, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,T,tol_state", [("tiny2", 40, 1e-4), ("tiny3", 30, 1e-4), ("C2", 100, 1e-3),
                                              ("C3", 60, 1e-3)])
def test_fcr_state_and_gradients_vs_oracle(name, T, tol_state):
    if name == "tiny2":
        sc = scenes.tiny(2, seed=61, res=32, n_cells=(8, 8), steps=T, K=2, s=40.0)
    elif name == "tiny3":
        sc = scenes.tiny(3, seed=62, res=32, n_cells=(6, 6, 6), steps=T, K=2, s=40.0)
    else:
        sc = scenes.CONFIGS[name](steps=T)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, material=1))
    sim.set_scene(sc)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    cfg = oracle_cfg(sc, material=1)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    ox, ov, oC, oF = oracle.unpack(traj[T], sc.dim)
    for k, a, b in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC)):
        assert rel_err(a, b) < tol_state, (k, rel_err(a, b))
    rng = np.random.default_rng(5)
    w = rng.standard_normal(traj[T].shape)
    wx, wv, wC, wF = oracle.unpack(w, sc.dim)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    g0, gE, gnu, ga = oracle.backward(cfg, traj, m, vol, E, nu, aid, act[:T], w)
    gx, gv, gC, gF = oracle.unpack(g0, sc.dim)
    assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF), ("dC0", g["dC0"], gC),
                  ("dE", g["dE"], gE), ("dnu", g["dnu"], gnu), ("da", g["da"][0, :T], ga)])


def test_fcr_one_step_tight():
    """One step: state within the north_star's 1e-5."""
    sc = scenes.tiny(3, seed=63, res=32, n_cells=(6, 6, 6), steps=1, K=2, s=40.0)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=1, material=1))
    sim.set_scene(sc)
    sim.forward(1)
    cfg = oracle_cfg(sc, material=1)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:1], 1)
    for a, b in zip(sim.get_state(1), (lambda u: (u[0], u[1], u[3], u[2]))(oracle.unpack(traj[1], 3))):
        assert rel_err(a, b) < 1e-5


def _rotations(n, d, rng):
    """n random proper rotations (QR of a Gaussian, sign-fixed, det +1)."""
    Q = np.empty((n, d, d))
    for p in range(n):
        q, r = np.linalg.qr(rng.standard_normal((d, d)))
        q = q * np.sign(np.diag(r))
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        Q[p] = q
    return Q


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("kind", ["rotation", "equal_stretch"])
@pytest.mark.parametrize("material", [0, 1])
def test_degenerate_deformation_gradients(d, kind, material):
    """F0 with repeated singular values -- pure rotations (F F^T = I: every stretch equal) and
    R diag(1.1, 1.1[, 0.9]) (a repeated pair) -- the degenerate inputs of the fixed-corotated
    eigen-decomposition and of its Lyapunov-solve adjoint (R21); neo-Hookean alongside.  The
    GPU's Jacobi route and the oracle's polar decomposition must agree on state and gradients."""
    T = 3
    sc = scenes.tiny(d, seed=63 + d, res=32, n_cells=(5,) * d, steps=T, K=2, s=30.0)
    rng = np.random.default_rng(64 + d)
    n = sc.n
    R = _rotations(n, d, rng)
    if kind == "equal_stretch":
        S = np.diag([1.1, 1.1, 0.9][:d])
        R = R @ S @ np.transpose(_rotations(n, d, rng), (0, 2, 1))
    sc.F = R[None].astype(np.float32)
    sc.C = np.zeros_like(sc.C)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, material=material))
    sim.set_scene(sc)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    cfg = oracle_cfg(sc, material=material)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    for k, a, b in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC)):
        assert rel_err(a, b) < 1e-4, (k, rel_err(a, b))
    w = np.random.default_rng(65).standard_normal(traj[T].shape)
    wx, wv, wC, wF = oracle.unpack(w, d)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    g0, gE, gnu, ga = oracle.backward(cfg, traj, m, vol, E, nu, aid, act[:T], w)
    gx, gv, gC, gF = oracle.unpack(g0, d)
    assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF),
                  ("dC0", g["dC0"], gC), ("dE", g["dE"], gE), ("dnu", g["dnu"], gnu),
                  ("da", g["da"][0, :T], ga)])
