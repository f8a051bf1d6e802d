"""Pins of the oracle's fixed-corotated model (NEXT N3, DESIGN R21): SPEC's and
hand-evaluated stresses, polar-decomposition examples, P = FD of psi, Hessian = FD of P and
major-symmetric, rotation equivariance, and the whole reverse pass vs central FD."""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
from paper_1810_01054_b200 import scenes
from tests.helpers import ang_mom, oracle_cfg, oracle_params, oracle_state


def _rot2(th):
    return np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])


def _rand_F(d, rng, lo=0.6, hi=1.6):
    """F = U diag(s) V^T with singular values in [lo, hi] and det > 0."""
    if d == 2:
        U, V = _rot2(rng.uniform(0, 6.3)), _rot2(rng.uniform(0, 6.3))
    else:
        U = Rotation.random(random_state=int(rng.integers(1 << 30))).as_matrix()
        V = Rotation.random(random_state=int(rng.integers(1 << 30))).as_matrix()
    return U @ np.diag(rng.uniform(lo, hi, d)) @ V.T


def test_spec_stress_examples():
    # SPEC S:135-137 (2D) and their 3D analogues, hand-evaluated
    np.testing.assert_array_equal(oracle.pk1(np.eye(2), 3.0, 5.0, 1), np.zeros((2, 2)))
    np.testing.assert_allclose(oracle.pk1(np.diag([2.0, 1.0]), 1.0, 0.0, 1), np.diag([2.0, 0.0]), atol=1e-15)
    np.testing.assert_allclose(oracle.pk1(np.diag([2.0, 1.0]), 0.0, 1.0, 1), np.diag([1.0, 2.0]), atol=1e-15)
    np.testing.assert_allclose(oracle.pk1(np.eye(3), 3.0, 5.0, 1), np.zeros((3, 3)), atol=1e-15)
    np.testing.assert_allclose(oracle.pk1(np.diag([2.0, 1.0, 1.0]), 1.0, 0.0, 1), np.diag([2.0, 0, 0]), atol=1e-14)
    np.testing.assert_allclose(oracle.pk1(np.diag([2.0, 1.0, 1.0]), 0.0, 1.0, 1), np.diag([1.0, 2.0, 2.0]), atol=1e-14)
    # psi at a pure stretch: mu sum (s - 1)^2 + lam/2 (J - 1)^2
    assert abs(oracle.psi(np.diag([1.5, 0.8, 1.1]), 2.0, 3.0, 1)
               - (2.0 * (0.25 + 0.04 + 0.01) + 1.5 * (1.5 * 0.8 * 1.1 - 1) ** 2)) < 1e-14


def test_polar_examples():
    # SPEC S:127-129
    np.testing.assert_allclose(oracle.polar(np.eye(2)), np.eye(2), atol=1e-15)
    np.testing.assert_allclose(oracle.polar(_rot2(0.7) @ np.diag([1.5, 0.4])), _rot2(0.7), atol=1e-14)
    np.testing.assert_allclose(oracle.polar(np.diag([2.0, 1.0])), np.eye(2), atol=1e-15)
    rng = np.random.default_rng(3)
    for _ in range(20):
        Q = Rotation.random(random_state=int(rng.integers(1 << 30))).as_matrix()
        U = Rotation.random(random_state=int(rng.integers(1 << 30))).as_matrix()
        S = U @ np.diag(rng.uniform(0.5, 2.0, 3)) @ U.T
        np.testing.assert_allclose(oracle.polar(Q @ S), Q, atol=1e-12)
    with pytest.raises(oracle.OracleError):
        oracle.polar(np.diag([1.0, 1.0, -1.0]))


@pytest.mark.parametrize("d", [2, 3])
def test_P_is_gradient_of_psi_and_hessian_of_P(d):
    rng = np.random.default_rng(10 + d)
    h = 1e-6
    for _ in range(25):
        F = _rand_F(d, rng)
        mu, lam = rng.uniform(0.5, 2), rng.uniform(0.5, 2)
        P = oracle.pk1(F, mu, lam, 1)
        H = oracle.dPdF(F, mu, lam, 1)
        num = np.zeros((d, d))
        numH = np.zeros((d, d, d, d))
        for a in range(d):
            for b in range(d):
                Fp, Fm = F.copy(), F.copy()
                Fp[a, b] += h
                Fm[a, b] -= h
                num[a, b] = (oracle.psi(Fp, mu, lam, 1) - oracle.psi(Fm, mu, lam, 1)) / (2 * h)
                numH[:, :, a, b] = (oracle.pk1(Fp, mu, lam, 1) - oracle.pk1(Fm, mu, lam, 1)) / (2 * h)
        np.testing.assert_allclose(P, num, rtol=1e-7, atol=1e-8)
        np.testing.assert_allclose(H, numH, rtol=1e-6, atol=1e-7)
        # Hessian of psi: major symmetry
        np.testing.assert_allclose(H, H.transpose(2, 3, 0, 1), atol=1e-12)


@pytest.mark.parametrize("d", [2, 3])
def test_rotation_equivariance_and_symmetric_kirchhoff(d):
    rng = np.random.default_rng(20 + d)
    for _ in range(20):
        F = _rand_F(d, rng)
        Q = _rot2(rng.uniform(0, 6.3)) if d == 2 else Rotation.random(random_state=int(rng.integers(1 << 30))).as_matrix()
        P = oracle.pk1(F, 1.3, 0.7, 1)
        np.testing.assert_allclose(oracle.pk1(Q @ F, 1.3, 0.7, 1), Q @ P, atol=1e-12)
        tau = P @ F.T
        np.testing.assert_allclose(tau, tau.T, atol=1e-12)


@pytest.mark.parametrize("d", [2, 3])
def test_fcr_step_conserves_momentum_and_angular_momentum(d):
    """With g = 0, no walls touched, fixed-corotated stress + actuation: linear momentum and
    the APIC-augmented angular momentum are conserved by the step (tau symmetric)."""
    sc = scenes.tiny(d, seed=70 + d, res=16, K=2, s=60.0, steps=3, perturb=True)
    cfg = oracle_cfg(sc, gravity=(0.0,) * d, material=1)
    m, vol, E, nu, aid, act = oracle_params(sc)
    st = oracle_state(sc)
    traj = oracle.forward(cfg, st, m, vol, E, nu, aid, act, 3)
    dx = 1.0 / sc.res
    for t in range(1, 4):
        x, v, Cm, F = oracle.unpack(traj[t], d)
        x0, v0, C0, F0 = oracle.unpack(traj[0], d)
        np.testing.assert_allclose((m[:, None] * v).sum(0), (m[:, None] * v0).sum(0), atol=1e-12)
        np.testing.assert_allclose(ang_mom(x, v, Cm, m, dx), ang_mom(x0, v0, C0, m, dx), atol=1e-12)


@pytest.mark.parametrize("d", [2, 3])
def test_fcr_gradients_vs_central_fd(d):
    """Reverse mode with the fixed-corotated Hessian (steps A-L) against central differences
    on sampled state entries, E, nu and actuation; floor friction + actuation, 8 steps."""
    T = 8
    res = 16
    center = [res // 2 - 1] * d
    center[1] = 3
    sc = scenes.tiny(d, seed=80 + d, res=res, n_cells=(3,) * d, K=2, s=60.0, steps=T, center=tuple(center))
    cfg = oracle_cfg(sc, friction=(0.3, 0.0, 0.6, 0.0, 0.0, 0.0), material=1)
    m, vol, E, nu, aid, act = oracle_params(sc)
    st = oracle_state(sc)
    rng = np.random.default_rng(90 + d)
    w = rng.standard_normal(st.shape)

    def L(st_=st, E_=E, nu_=nu, act_=act):
        return float(np.sum(oracle.forward(cfg, st_, m, vol, E_, nu_, aid, act_, T)[-1] * w))

    traj = oracle.forward(cfg, st, m, vol, E, nu, aid, act, T)
    g0, gE, gnu, ga = oracle.backward(cfg, traj, m, vol, E, nu, aid, act, w)
    scale = max(np.abs(g0).max(), np.abs(gE).max(), np.abs(gnu).max(), np.abs(ga).max())

    def check(num, ana, what):
        assert abs(num - ana) <= 1e-6 * max(abs(num), 1e-3 * scale), (what, num, ana)

    for _ in range(30):
        p, c = rng.integers(sc.n), rng.integers(st.shape[1])
        h = 1e-6 if c < d else (1e-5 if c < 2 * d else (1e-4 if c < 2 * d + d * d else 1e-5))  # x, v, C, F
        sp, sm = st.copy(), st.copy()
        sp[p, c] += h
        sm[p, c] -= h
        check((L(st_=sp) - L(st_=sm)) / (2 * h), g0[p, c], f"state[{p},{c}]")
    for _ in range(6):
        p = rng.integers(sc.n)
        Ep, Em = E.copy(), E.copy()
        Ep[p] += 1e-3
        Em[p] -= 1e-3
        check((L(E_=Ep) - L(E_=Em)) / 2e-3, gE[p], f"E[{p}]")
        np_, nm = nu.copy(), nu.copy()
        np_[p] += 1e-7
        nm[p] -= 1e-7
        check((L(nu_=np_) - L(nu_=nm)) / 2e-7, gnu[p], f"nu[{p}]")
    for _ in range(6):
        t, k, a = rng.integers(T), rng.integers(cfg.n_act), rng.integers(d)
        ap, am = act.copy(), act.copy()
        ap[t, k, a] += 1e-5
        am[t, k, a] -= 1e-5
        check((L(act_=ap) - L(act_=am)) / 2e-5, ga[t, k, a], f"a[{t},{k},{a}]")
