"""Pins of the oracle's forward step against conservation laws and closed forms (P:123-126
Eqs. 1-2 as invariants; SURVEY.md 8c "What pins each part").  CPU only, fp64."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import scenes
from tests.helpers import ang_mom, oracle_cfg, oracle_params, oracle_state, run_oracle


def _no_walls(scene):
    return oracle_cfg(scene, gravity=(0.0, 0.0, 0.0), friction=(0.0,) * 6)


@pytest.mark.parametrize("d", [2, 3])
def test_mass_and_momentum_through_p2g(d):
    """Sum_i m_i = Sum_p m_p (Eq. 3); Sum_i p_i = Sum_p m_p v_p (Eq. 5) for ANY stress,
    affine C and actuation, because Sum_i N (x_i - x_p) = 0."""
    sc = scenes.tiny(d, seed=21, res=16, K=2, s=80.0)
    cfg = _no_walls(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    st = oracle_state(sc)
    mi, pi, _, _ = oracle.step_grid(cfg, st, m, vol, E, nu, aid, act[0])
    x, v, _, _ = oracle.unpack(st, d)
    assert abs(mi.sum() - m.sum()) < 1e-14 * m.sum()
    np.testing.assert_allclose(pi.sum(0), (m[:, None] * v).sum(0), atol=1e-14 * np.abs(v).max() * m.sum())


@pytest.mark.parametrize("d", [2, 3])
def test_momentum_and_angular_momentum_one_step(d):
    """No gravity, no wall contact: one whole step (stress, actuation, random C) conserves
    linear momentum and the augmented APIC angular momentum (tau symmetric)."""
    sc = scenes.tiny(d, seed=22, res=16, K=2, s=80.0)
    cfg = _no_walls(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act, 3)
    dx = 1.0 / sc.res
    P0 = None
    L0 = None
    for t in range(4):
        x, v, Cm, F = oracle.unpack(traj[t], d)
        P = (m[:, None] * v).sum(0)
        L = ang_mom(x, v, Cm, m, dx)
        if t == 0:
            P0, L0 = P, L
        else:
            np.testing.assert_allclose(P, P0, atol=1e-13 * np.abs(P0).max() + 1e-18)
            np.testing.assert_allclose(L, L0, rtol=1e-10, atol=1e-14 * (np.abs(L0).max() + 1e-12))


@pytest.mark.parametrize("d", [2, 3])
def test_rigid_rotation_preserved(d):
    """v = w x (x - xc), C = [w]x, F = I (stress free): one step reproduces v and C exactly
    (APIC + the quadratic kernel's D = dx^2/4 I)."""
    sc = scenes.tiny(d, seed=23, res=16, K=0, perturb=False)
    cfg = _no_walls(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    x = sc.x[0].astype(np.float64)
    xc = x.mean(0)
    if d == 2:
        w = 1.7
        W = np.array([[0.0, -w], [w, 0.0]])
    else:
        wv = np.array([0.3, -1.1, 0.8])
        W = np.array([[0, -wv[2], wv[1]], [wv[2], 0, -wv[0]], [-wv[1], wv[0], 0]])
    v = (x - xc) @ W.T
    Cm = np.broadcast_to(W, (x.shape[0], d, d))
    st = oracle.pack(x, v, Cm, np.broadcast_to(np.eye(d), (x.shape[0], d, d)))
    traj = oracle.forward(cfg, st, m, vol, E, nu, None, None, 1)
    x1, v1, C1, F1 = oracle.unpack(traj[1], d)
    np.testing.assert_allclose(v1, v, atol=1e-13)
    np.testing.assert_allclose(C1, Cm, atol=1e-11)
    np.testing.assert_allclose(F1, np.broadcast_to(np.eye(d) + cfg.dt * W, F1.shape), atol=1e-13)


@pytest.mark.parametrize("d", [2, 3])
def test_uniform_translation(d):
    """Uniform v, C = 0, F = I: v' = v, C' = 0, F' = F."""
    sc = scenes.tiny(d, seed=24, res=16, K=0, perturb=False)
    cfg = _no_walls(sc)
    m, vol, E, nu, _, _ = oracle_params(sc)
    n = sc.n
    v = np.tile(np.linspace(0.3, -0.7, d), (n, 1))
    st = oracle.pack(sc.x[0], v, np.zeros((n, d, d)), np.broadcast_to(np.eye(d), (n, d, d)))
    traj = oracle.forward(cfg, st, m, vol, E, nu, None, None, 1)
    x1, v1, C1, F1 = oracle.unpack(traj[1], d)
    np.testing.assert_allclose(v1, v, atol=1e-14)
    np.testing.assert_allclose(C1, 0, atol=1e-11)
    np.testing.assert_allclose(F1, np.broadcast_to(np.eye(d), F1.shape), atol=1e-14)
    np.testing.assert_allclose(x1,sc.x[0] + cfg.dt * v, atol=1e-15)


def test_com_closed_form_with_gravity():
    """Without wall contact, CoM_n = CoM_0 + dt sum_{k=1..n} (P_0/M + k dt g) exactly, for any
    internal stress and actuation (C1 scene, 50 steps)."""
    sc = scenes.block_2d(steps=50, perturb=True)
    cfg, traj = run_oracle(sc)
    m = sc.mass[0].astype(np.float64)
    M = m.sum()
    x0, v0, _, _ = oracle.unpack(traj[0], 2)
    com0 = (m[:, None] * x0).sum(0) / M
    P0 = (m[:, None] * v0).sum(0)
    g = np.array(cfg.gravity[:2])
    for t in (1, 10, 50):
        xt = oracle.unpack(traj[t], 2)[0]
        com = (m[:, None] * xt).sum(0) / M
        exp = com0 + cfg.dt * sum(P0 / M + k * cfg.dt * g for k in range(1, t + 1))
        np.testing.assert_allclose(com, exp, atol=1e-14)


def test_errors_out_of_domain_and_inverted():
    sc = scenes.tiny(3, seed=25, res=16, K=0)
    cfg = oracle_cfg(sc)
    m, vol, E, nu, _, _ = oracle_params(sc)
    st = oracle_state(sc)
    bad = st.copy()
    bad[0, 0] = 0.01  # base = -1
    with pytest.raises(oracle.OracleError) as e:
        oracle.forward(cfg, bad, m, vol, E, nu, None, None, 1)
    assert e.value.code == oracle.ORC_ERR_OUT_OF_DOMAIN
    inv = st.copy()
    inv[1, 2 * 3 + 9:] = np.diag([-1.0, 1.0, 1.0]).reshape(-1)
    with pytest.raises(oracle.OracleError) as e:
        oracle.forward(cfg, inv, m, vol, E, nu, None, None, 1)
    assert e.value.code == oracle.ORC_ERR_INVERTED


# ---- binning ----------------------------------------------------------------------------
def test_binning_golden():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "binning.txt")
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        t = line.split()
        dim, res, r = int(t[0]), int(t[1]), int(t[2])
        x = np.array([float(s) for s in t[3:3 + dim]], np.float32)
        B = r + 1
        xs = np.tile(np.full(dim, 0.5, np.float32), (B, 1, 1))
        xs[r, 0] = x
        key, perm, bs = oracle.bin_particles(dim, res, xs)
        assert key[r] == int(t[3 + dim])


@pytest.mark.parametrize("d", [2, 3])
def test_binning_brute_force(d):
    """Stable sort by key against an O(n^2) brute-force ranking on tiny inputs, including
    ties (many particles per cell) and several rollouts."""
    rng = np.random.default_rng(26)
    res, B, n = 32, 3, 200
    x = rng.uniform(2.0 / res, 1 - 3.0 / res, (B, n, d)).astype(np.float32)
    x[:, :50] = x[:, :1]  # exact ties
    key, perm, bs = oracle.bin_particles(d, res, x)
    tot = B * n
    rank = np.array([sum(1 for q in range(tot) if key[q] < key[p] or (key[q] == key[p] and q < p))
                     for p in range(tot)])
    expect = np.empty(tot, np.int64)
    expect[rank] = np.arange(tot)
    np.testing.assert_array_equal(perm, expect)
    Bb = 4 if d == 3 else 8
    cpb = Bb ** d
    blocks = key // cpb
    for gb in range(0, len(bs) - 1, 7):
        assert bs[gb] == np.sum(blocks < gb)
    assert bs[-1] == tot
