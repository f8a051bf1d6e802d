"""Pins of the oracle's reverse mode (steps A-L, chained per P:165) against the
exact closed-form CoM gradient (A1 analogue), the frictionless-wall tangential
gradient (A2 analogue) and central finite differences in fp64 (cases B/C style,
P:225-226).  CPU only."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import scenes
from tests.helpers import oracle_cfg, oracle_params, oracle_state, rel_err


def _loss_seed(n, d, w_rec):
    return w_rec


def _com_seed(m, d, axis, n):
    S = oracle.S_of(d)
    seed = np.zeros((n, S))
    seed[:, axis] = m / m.sum()
    return seed


@pytest.mark.parametrize("d,T", [(2, 50), (3, 20), (2, 1000)])
def test_com_gradient_closed_form(d, T):
    """L = CoM_x(T).  Without wall contact CoM_T = CoM_0 + dt sum_k (P_0/M + k dt g) for any
    stress, actuation and internal collision, so dL/dx0_p = m_p/M e_x, dL/dv0_p = T dt m_p/M
    e_x and dL/dF0 = dL/dC0 = dL/dE = dL/dnu = dL/da = 0 exactly (SURVEY 8c, A1 analogue;
    T = 1000 is the long-horizon stability case)."""
    sc = scenes.tiny(d, seed=31 + d, res=16 if d == 2 else 16, K=2, s=40.0, steps=T,
                     center=(6,) * d, v0=None)
    cfg = oracle_cfg(sc, friction=(0.0,) * 6)
    # keep away from walls: tiny v, and gravity kept (it does not break the closed form)
    m, vol, E, nu, aid, act = oracle_params(sc)
    st = oracle_state(sc)
    st[:, d:2 * d] *= 0.05
    traj = oracle.forward(cfg, st, m, vol, E, nu, aid, act, T)
    xs = traj[:, :, :d]
    assert xs.min() > 3.5 / sc.res and xs.max() < 1 - 4.5 / sc.res, "scene touched a wall band"
    seed = _com_seed(m, d, 0, sc.n)
    g0, gE, gnu, ga = oracle.backward(cfg, traj, m, vol, E, nu, aid, act, seed)
    gx, gv, gC, gF = oracle.unpack(g0, d)
    ex = np.zeros(d)
    ex[0] = 1.0
    M = m.sum()
    np.testing.assert_allclose(gx, (m / M)[:, None] * ex, atol=1e-11 / sc.n)
    np.testing.assert_allclose(gv, (T * cfg.dt * m / M)[:, None] * ex, atol=1e-13 * T / sc.n)
    scale = 1.0 / sc.n
    assert np.abs(gC).max() < 1e-12 * scale * T
    assert np.abs(gF).max() < 1e-11 * scale * T
    assert np.abs(gE).max() < 1e-14 * T
    assert np.abs(gnu).max() < 1e-11 * T
    assert np.abs(ga).max() < 1e-13 * T


def _fd_scene(d, seed, T, friction=(0.3, 0.0, 0.6, 0.0, 0.0, 0.0), floor=True):
    res = 16
    nc = (3,) * d
    center = [res // 2 - 1] * d
    if floor:
        center[1] = 3  # cells 3.. -> nodes reach the floor band (< 3)
    sc = scenes.tiny(d, seed=seed, res=res, n_cells=nc, K=2, s=60.0, steps=T, center=tuple(center))
    cfg = oracle_cfg(sc, friction=friction)
    return sc, cfg


def _forward_loss(cfg, st, m, vol, E, nu, aid, act, w, T):
    traj = oracle.forward(cfg, st, m, vol, E, nu, aid, act, T)
    return float(np.sum(traj[-1] * w)), traj


@pytest.mark.parametrize("d", [2, 3])
def test_gradients_vs_central_fd(d):
    """Random linear loss on the final state; every input family (x0, v0, C0, F0, E, nu, a)
    against central differences on sampled coordinates.  Scene touches the floor band with
    friction (step L), actuation on, random F0/C0 (SURVEY 8d parity recipe)."""
    T = 8
    sc, cfg = _fd_scene(d, 40 + d, T)
    m, vol, E, nu, aid, act = oracle_params(sc)
    st = oracle_state(sc)
    rng = np.random.default_rng(50 + d)
    w = rng.standard_normal(st.shape)
    L0, traj = _forward_loss(cfg, st, m, vol, E, nu, aid, act, w, T)
    g0, gE, gnu, ga = oracle.backward(cfg, traj, m, vol, E, nu, aid, act, w)

    def fd(fun, h):
        return (fun(h) - fun(-h)) / (2 * h)

    errs = []
    # state coordinates
    S = st.shape[1]
    for _ in range(60):
        p, c = rng.integers(sc.n), rng.integers(S)
        scale = 1e-3 if c < d else (1e-2 if c < 2 * d else 1e-2)

        def f(h):
            s2 = st.copy()
            s2[p, c] += h
            return _forward_loss(cfg, s2, m, vol, E, nu, aid, act, w, T)[0]
        num = fd(f, 1e-6 * scale / 1e-3 * 1e-1)
        errs.append((abs(num - g0[p, c]), abs(num), f"state[{p},{c}]"))
    for _ in range(10):
        p = rng.integers(sc.n)

        def fE(h):
            E2 = E.copy(); E2[p] += h
            return _forward_loss(cfg, st, m, vol, E2, nu, aid, act, w, T)[0]

        def fn(h):
            n2 = nu.copy(); n2[p] += h
            return _forward_loss(cfg, st, m, vol, E, n2, aid, act, w, T)[0]
        num = fd(fE, 1e-3)
        errs.append((abs(num - gE[p]), abs(num), f"E[{p}]"))
        num = fd(fn, 1e-7)
        errs.append((abs(num - gnu[p]), abs(num), f"nu[{p}]"))
    for _ in range(10):
        t, k, a = rng.integers(T), rng.integers(cfg.n_act), rng.integers(d)

        def fa(h):
            a2 = act.copy(); a2[t, k, a] += h
            return _forward_loss(cfg, st, m, vol, E, nu, aid, a2, w, T)[0]
        num = fd(fa, 1e-5)
        errs.append((abs(num - ga[t, k, a]), abs(num), f"a[{t},{k},{a}]"))
    gmax = max(np.abs(g0).max(), np.abs(gE).max(), np.abs(gnu).max(), np.abs(ga).max())
    bad = [(e, n, s) for e, n, s in errs if e > 1e-6 * max(n, 1e-3 * gmax)]
    assert not bad, bad[:5]


@pytest.mark.parametrize("d", [2, 3])
def test_dot_product(d):
    """(dL/ds0) . dir = directional central difference along a random direction of ALL
    inputs at once, 20 steps with floor contact."""
    T = 20
    sc, cfg = _fd_scene(d, 60 + d, T)
    m, vol, E, nu, aid, act = oracle_params(sc)
    st = oracle_state(sc)
    rng = np.random.default_rng(70 + d)
    w = rng.standard_normal(st.shape)
    _, traj = _forward_loss(cfg, st, m, vol, E, nu, aid, act, w, T)
    g0, gE, gnu, ga = oracle.backward(cfg, traj, m, vol, E, nu, aid, act, w)
    ds = rng.standard_normal(st.shape) * np.concatenate([np.full(d, 1e-3), np.full(st.shape[1] - d, 1e-2)])
    dE = rng.standard_normal(E.shape) * 10.0
    dnu = rng.standard_normal(nu.shape) * 1e-3
    da = rng.standard_normal(act.shape) * 0.1
    pred = np.sum(g0 * ds) + np.sum(gE * dE) + np.sum(gnu * dnu) + np.sum(ga * da[:T])
    for h in (1e-4, 1e-5):
        Lp = _forward_loss(cfg, st + h * ds, m, vol, E + h * dE, nu + h * dnu, aid, act + h * da, w, T)[0]
        Lm = _forward_loss(cfg, st - h * ds, m, vol, E - h * dE, nu - h * dnu, aid, act - h * da, w, T)[0]
        num = (Lp - Lm) / (2 * h)
        assert abs(num - pred) < 1e-6 * abs(pred), (h, num, pred)


def test_frictionless_wall_tangential_gradient():
    """A2 analogue: a block slides into the frictionless +x wall (c = 0, g = 0).  Step
    L with c = 0 keeps every node's tangential velocity, so CoM_y(T) = CoM_y(0) + T dt
    P_y(0)/M and dCoM_y(T)/dv0_{p,y} = T dt m_p / M exactly, bounce or not."""
    d, T = 2, 200
    res = 16
    sc = scenes.tiny(d, seed=80, res=res, K=0, steps=T, perturb=True, center=(10, 7))
    cfg = oracle_cfg(sc, gravity=(0.0, 0.0), friction=(0.0,) * 6)
    m, vol, E, nu, aid, act = oracle_params(sc)
    st = oracle_state(sc)
    st[:, 0 + d] += 1.0   # v_x toward the +x wall
    st[:, 1 + d] += 0.1
    traj = oracle.forward(cfg, st, m, vol, E, nu, aid, act, T)
    x = traj[:, :, :d]
    assert x[:, :, 0].max() * res > res - 4.5, "block never reached the +x band"
    assert x[:, :, 1].min() * res > 3.5 and x[:, :, 1].max() * res < res - 4.5
    M = m.sum()
    com_y = (traj[:, :, 1] * m).sum(1) / M
    Py0 = (st[:, 1 + d] * m).sum()
    np.testing.assert_allclose(com_y[-1], com_y[0] + T * cfg.dt * Py0 / M, atol=1e-13)
    seed = _com_seed(m, d, 1, sc.n)
    g0, gE, gnu, ga = oracle.backward(cfg, traj, m, vol, E, nu, aid, act, seed)
    np.testing.assert_allclose(g0[:, 1 + d], T * cfg.dt * m / M, rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(g0[:, 1], m / M, rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("d", [2, 3])
def test_mass_gradient_and_running_loss_vs_fd(d):
    """NEXT N3 (dL/dm_p, the gradient behind the paper's density inference) and N4
    (a running loss L = sum_t <w_t, state_t>): oracle reverse mode vs central differences on
    sampled masses and along a random direction of the initial state."""
    T = 8
    sc, cfg = _fd_scene(d, 90 + d, T)
    m, vol, E, nu, aid, act = oracle_params(sc)
    st = oracle_state(sc)
    rng = np.random.default_rng(91 + d)
    W = rng.standard_normal((T + 1,) + st.shape)

    def L(st_, m_):
        traj = oracle.forward(cfg, st_, m_, vol, E, nu, aid, act, T)
        return float(np.sum(traj * W)), traj

    L0, traj = L(st, m)
    g0, gE, gnu, ga, gm = oracle.backward_ex(cfg, traj, m, vol, E, nu, aid, act, W)
    for p in rng.choice(sc.n, 8, replace=False):
        h = 1e-6 * m[p]
        mp, mm = m.copy(), m.copy()
        mp[p] += h
        mm[p] -= h
        fd = (L(st, mp)[0] - L(st, mm)[0]) / (2 * h)
        assert abs(fd - gm[p]) < 1e-5 * max(abs(fd), 1e-3 * np.abs(gm).max()), (p, fd, gm[p])
    ds = rng.standard_normal(st.shape) * np.concatenate([np.full(d, 1e-3), np.full(st.shape[1] - d, 1e-2)])
    pred = float(np.sum(g0 * ds))
    h = 1e-4
    fd = (L(st + h * ds, m)[0] - L(st - h * ds, m)[0]) / (2 * h)
    assert abs(fd - pred) < 1e-6 * abs(pred), (fd, pred)
    # the running loss reduces to orc_backward when only the last seed is non-zero
    W2 = np.zeros_like(W)
    W2[-1] = W[-1]
    a = oracle.backward_ex(cfg, traj, m, vol, E, nu, aid, act, W2)
    b = oracle.backward(cfg, traj, m, vol, E, nu, aid, act, W[-1])
    np.testing.assert_array_equal(a[0], b[0])
