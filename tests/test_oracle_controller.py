"""Pins of the controller oracle (NEXT N1, SPEC observe/act/controller_adjoint S:377-408):
SPEC's worked examples, the reduction to the open-loop oracle when W = 0, tanh saturation,
and central finite differences in fp64 of a closed-loop loss w.r.t. W, b, target, x0, v0."""
import numpy as np
import pytest

import oracle
from oracle import controller as ctl
from paper_1810_01054_b200 import scenes
from tests.helpers import oracle_cfg, oracle_params, oracle_state


def test_observe_spec_examples():
    # one group, two equal-mass particles at (0,0), (2,0), v = 0, target (5,5) -> (5,5, 1,0, 0,0)
    z = ctl.observe(np.array([[0.0, 0.0], [2.0, 0.0]]), np.zeros((2, 2)), np.ones(2), np.zeros(2, int), 1,
                    (5.0, 5.0))
    np.testing.assert_array_equal(z, [5, 5, 1, 0, 0, 0])
    # unequal masses 1 at (0,0), 3 at (4,0) -> CoM (3,0)
    z = ctl.observe(np.array([[0.0, 0.0], [4.0, 0.0]]), np.zeros((2, 2)), np.array([1.0, 3.0]),
                    np.zeros(2, int), 1, (0.0, 0.0))
    np.testing.assert_allclose(z[2:4], [3.0, 0.0], rtol=0, atol=1e-15)
    # translation equivariance of the CoM slots, velocity slots untouched
    rng = np.random.default_rng(0)
    x, v, m = rng.random((20, 3)), rng.random((20, 3)), rng.random(20) + 0.5
    aid = np.arange(20) % 2
    s = np.array([0.25, -0.5, 0.125])
    z0 = ctl.observe(x, v, m, aid, 2, np.zeros(3))
    z1 = ctl.observe(x + s, v, m, aid, 2, np.zeros(3))
    np.testing.assert_allclose(z1[3:9] - z0[3:9], np.tile(s, 2), atol=1e-14)
    np.testing.assert_array_equal(z1[9:], z0[9:])
    with pytest.raises(ValueError):
        ctl.observe(x, v, m, aid, 3, np.zeros(3))  # group 2 is empty


def test_act_spec_examples():
    assert np.all(ctl.act(np.zeros((4, 6)), np.zeros(4), np.ones(6)) == 0.0)
    assert np.all(np.abs(ctl.act(np.zeros((4, 6)), np.full(4, 20.0), np.ones(6)) - 1.0) < 1e-15)
    z = np.random.default_rng(1).uniform(-1e-3, 1e-3, 5)
    np.testing.assert_allclose(ctl.act(np.eye(5), np.zeros(5), z), z - z ** 3 / 3, rtol=0, atol=1e-9)


def _scene(d, seed, T):
    sc = scenes.tiny(d, seed=seed, res=16, n_cells=(3,) * d, K=2, s=60.0, steps=T,
                     center=(6, 3) if d == 2 else (6, 3, 6))
    cfg = oracle_cfg(sc, friction=(0.3, 0.0, 0.6, 0.0, 0.0, 0.0))
    return sc, cfg


@pytest.mark.parametrize("d", [2, 3])
def test_zero_W_is_open_loop_tanh_b(d):
    """W = 0 makes a_t = tanh(b) for every t: the closed-loop rollout is the open-loop rollout
    of that actuation, and dL/db = sum_t dL/da_t * (1 - tanh(b)^2) with the open-loop dL/da."""
    T = 6
    sc, cfg = _scene(d, 3 + d, T)
    m, vol, E, nu, aid, _ = oracle_params(sc)
    st = oracle_state(sc)
    K = cfg.n_act
    nz = ctl.n_obs(d, K)
    b = np.random.default_rng(4).uniform(-1, 1, K * d)
    traj, acts, zs = ctl.forward(cfg, st, m, vol, E, nu, aid, np.zeros((K * d, nz)), b, np.zeros(d), T)
    open_act = np.tile(np.tanh(b).reshape(1, K, d), (T, 1, 1))
    traj_o = oracle.forward(cfg, st, m, vol, E, nu, aid, open_act, T)
    np.testing.assert_array_equal(traj, traj_o)
    w = np.random.default_rng(5).standard_normal(st.shape)
    g, gE, gnu, gW, gb, gt, ga = ctl.backward(cfg, traj, m, vol, E, nu, aid, np.zeros((K * d, nz)), b, acts,
                                              zs, w)
    g_o, gE_o, gnu_o, ga_o = oracle.backward(cfg, traj_o, m, vol, E, nu, aid, open_act, w)
    np.testing.assert_allclose(g, g_o, rtol=1e-12, atol=1e-14 * np.abs(g_o).max())
    np.testing.assert_allclose(gb, (ga_o.reshape(T, -1) * (1 - np.tanh(b) ** 2)).sum(0), rtol=1e-10)
    np.testing.assert_array_equal(gt, 0.0)


@pytest.mark.parametrize("d", [2, 3])
def test_controller_gradients_vs_central_fd(d):
    """Closed loop (z depends on the state every step): dL/dW, dL/db, dL/dtarget and dL/dx0,
    dL/dv0 against central differences of L = <w, state_T> in fp64 (SPEC: finger-controller
    case C)."""
    T = 8
    sc, cfg = _scene(d, 10 + d, T)
    m, vol, E, nu, aid, _ = oracle_params(sc)
    st = oracle_state(sc)
    K = cfg.n_act
    nz = ctl.n_obs(d, K)
    rng = np.random.default_rng(20 + d)
    W = rng.standard_normal((K * d, nz)) * 0.5
    b = rng.uniform(-0.5, 0.5, K * d)
    target = np.array([0.7, 0.3, 0.5][:d])
    w = rng.standard_normal(st.shape)

    def L(W_=W, b_=b, t_=target, st_=st):
        traj = ctl.forward(cfg, st_, m, vol, E, nu, aid, W_, b_, t_, T)[0]
        return float(np.sum(traj[-1] * w))

    traj, acts, zs = ctl.forward(cfg, st, m, vol, E, nu, aid, W, b, target, T)
    g, gE, gnu, gW, gb, gt, ga = ctl.backward(cfg, traj, m, vol, E, nu, aid, W, b, acts, zs, w)
    assert np.abs(gW).max() > 1e-6 and np.abs(g[:, :d]).max() > 1e-6  # the loop is really closed

    def check(num, ana, what):
        assert abs(num - ana) <= 1e-6 * max(abs(num), 1e-3 * scale), (what, num, ana)

    scale = max(np.abs(gW).max(), np.abs(gb).max(), np.abs(g).max())
    h = 1e-6
    for _ in range(8):
        i, j = rng.integers(K * d), rng.integers(nz)
        Wp, Wm = W.copy(), W.copy()
        Wp[i, j] += h
        Wm[i, j] -= h
        check((L(W_=Wp) - L(W_=Wm)) / (2 * h), gW[i, j], f"W[{i},{j}]")
    for i in range(K * d):
        bp, bm = b.copy(), b.copy()
        bp[i] += h
        bm[i] -= h
        check((L(b_=bp) - L(b_=bm)) / (2 * h), gb[i], f"b[{i}]")
    for i in range(d):
        tp, tm = target.copy(), target.copy()
        tp[i] += h
        tm[i] -= h
        check((L(t_=tp) - L(t_=tm)) / (2 * h), gt[i], f"target[{i}]")
    for _ in range(8):
        p, c = rng.integers(sc.n), rng.integers(2 * d)  # x0 and v0 (the closed-loop paths)
        hp = 1e-7
        sp, sm = st.copy(), st.copy()
        sp[p, c] += hp
        sm[p, c] -= hp
        check((L(st_=sp) - L(st_=sm)) / (2 * hp), g[p, c], f"state[{p},{c}]")


def test_saturated_controller_has_no_parameter_gradient():
    """|Wz + b| >= 20 -> tanh' = 1 - a^2 < 1e-16: vanishing dL/dW, dL/db (SPEC example)."""
    T = 4
    sc, cfg = _scene(2, 30, T)
    m, vol, E, nu, aid, _ = oracle_params(sc)
    st = oracle_state(sc)
    K, d = cfg.n_act, 2
    nz = ctl.n_obs(d, K)
    W = np.zeros((K * d, nz))
    b = np.full(K * d, 25.0)
    traj, acts, zs = ctl.forward(cfg, st, m, vol, E, nu, aid, W, b, np.zeros(d), T)
    w = np.random.default_rng(31).standard_normal(st.shape)
    g, gE, gnu, gW, gb, gt, ga = ctl.backward(cfg, traj, m, vol, E, nu, aid, W, b, acts, zs, w)
    assert np.abs(ga).max() > 1e-8
    assert np.abs(gb).max() <= 1e-15 * np.abs(ga).max() * T
    assert np.abs(gW).max() <= 1e-15 * np.abs(ga).max() * T * np.abs(zs).max()
