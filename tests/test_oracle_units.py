"""Pins of the oracle's unit pieces against printed values, closed forms and finite
differences (never against the oracle itself).  CPU only."""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    out = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            out.append(line)
    return out


# ---- B-spline (R2) -------------------------------------------------------------------
def test_bspline_golden():
    for row in _rows("bspline.txt"):
        xg, base, w0, w1, w2 = row.split()
        b, w, _ = oracle.weights(float(xg))
        assert b == int(base)
        np.testing.assert_allclose(w, [float(w0), float(w1), float(w2)], rtol=0, atol=1e-15)


def test_bspline_moments():
    """Partition of unity, linear reproduction and the D_p = dx^2/4 I moment that makes the
    paper's 4/dx^2 factor the inverse inertia of this kernel."""
    rng = np.random.default_rng(1)
    for xg in rng.uniform(2.0, 60.0, 2000):
        b, w, _ = oracle.weights(xg)
        off = np.arange(3) + b - xg  # (x_i - x_p)/dx
        assert abs(w.sum() - 1.0) < 1e-14
        assert abs((w * off).sum()) < 1e-13
        assert abs((w * off * off).sum() - 0.25) < 1e-13
        assert np.all(w >= 0)


def test_bspline_derivative_fd():
    rng = np.random.default_rng(2)
    h = 1e-6
    for u in rng.uniform(-1.6, 1.6, 500):
        if min(abs(abs(u) - 0.5), abs(abs(u) - 1.5)) < 1e-4:
            continue
        fd = (oracle.N(u + h) - oracle.N(u - h)) / (2 * h)
        assert abs(fd - oracle.dN(u)) < 1e-8


# ---- constitutive model (R1) -----------------------------------------------------------
def test_stress_golden():
    for row in _rows("stress.txt"):
        lhs, rhs = row.split("|")
        vals = [float(t) for t in lhs.split()]
        dim, mu, lam = int(vals[0]), vals[1], vals[2]
        F = np.diag(vals[3:3 + dim])
        P = oracle.pk1(F, mu, lam)
        np.testing.assert_allclose(P, np.diag([float(t) for t in rhs.split()]), atol=1e-15)


def test_lame_golden():
    mu, lam = oracle.lame(1.0, 0.0)
    assert mu == 0.5 and lam == 0.0
    mu, lam = oracle.lame(2.5, 0.25)
    assert abs(mu - 1.0) < 1e-15 and abs(lam - 1.0) < 1e-15


def _rand_F(rng, d):
    return np.eye(d) + 0.25 * rng.standard_normal((d, d))


@pytest.mark.parametrize("d", [2, 3])
def test_pk1_is_gradient_of_psi(d):
    """P = d psi / dF by central differences of the textbook energy."""
    rng = np.random.default_rng(3 + d)
    h = 1e-6
    for _ in range(50):
        F = _rand_F(rng, d)
        if np.linalg.det(F) < 0.2:
            continue
        mu, lam = rng.uniform(0.1, 3.0, 2)
        P = oracle.pk1(F, mu, lam)
        fd = np.zeros((d, d))
        for a in range(d):
            for b in range(d):
                E = np.zeros((d, d))
                E[a, b] = h
                fd[a, b] = (oracle.psi(F + E, mu, lam) - oracle.psi(F - E, mu, lam)) / (2 * h)
        np.testing.assert_allclose(P, fd, atol=1e-7 * max(1, np.abs(P).max()))


@pytest.mark.parametrize("d", [2, 3])
def test_hessian_fd_and_symmetry(d):
    """d^2 psi / dF dF of step H = central differences of P; major symmetry."""
    rng = np.random.default_rng(7 + d)
    h = 1e-6
    for _ in range(30):
        F = _rand_F(rng, d)
        if np.linalg.det(F) < 0.2:
            continue
        mu, lam = rng.uniform(0.1, 3.0, 2)
        H = oracle.dPdF(F, mu, lam)
        for a in range(d):
            for b in range(d):
                E = np.zeros((d, d))
                E[a, b] = h
                fd = (oracle.pk1(F + E, mu, lam) - oracle.pk1(F - E, mu, lam)) / (2 * h)
                np.testing.assert_allclose(H[:, :, a, b], fd, atol=1e-6 * max(1, np.abs(H).max()))
        Hm = H.reshape(d * d, d * d)
        np.testing.assert_allclose(Hm, Hm.T, atol=1e-12 * np.abs(Hm).max())


def test_pk1_rotation_equivariance():
    rng = np.random.default_rng(11)
    for _ in range(50):
        F = _rand_F(rng, 3)
        if np.linalg.det(F) < 0.2:
            continue
        Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        if np.linalg.det(Q) < 0:
            Q[:, 0] *= -1
        mu, lam = rng.uniform(0.1, 3.0, 2)
        np.testing.assert_allclose(oracle.pk1(Q @ F, mu, lam), Q @ oracle.pk1(F, mu, lam),
                                   atol=1e-12)
        # tau = P F^T is symmetric for any F (what makes MLS forces torque free)
        P = oracle.pk1(F, mu, lam)
        tau = P @ F.T
        np.testing.assert_allclose(tau, tau.T, atol=1e-12)


# ---- step L ------------------------------------------------------------------
def test_projection_golden():
    for row in _rows("projection.txt"):
        c, vx, vy = (float(t) for t in row.split())
        out = oracle.project([1.0, -1.0], [0.0, 1.0], c)
        np.testing.assert_allclose(out, [vx, vy], atol=1e-9)


def test_projection_properties():
    rng = np.random.default_rng(12)
    for _ in range(300):
        v = rng.standard_normal(3)
        n = np.zeros(3)
        n[rng.integers(3)] = rng.choice([-1.0, 1.0])
        # c = 0 keeps the tangential velocity and removes only an inward normal component
        vs = oracle.project(v, n, 0.0)
        ln = v @ n
        vt = v - ln * n
        np.testing.assert_allclose(vs - (vs @ n) * n, vt, atol=1e-12)
        assert abs(vs @ n - max(ln, 0.0)) < 1e-12
        # sticky wall
        assert np.all(oracle.project(v, n, -1.0) == 0)
        # separating node: identity
        if ln >= 0:
            assert np.all(oracle.project(v, n, 0.7) == v)


def test_projection_adjoint_fd():
    """Adjoint P:622-634 equals the transposed Jacobian of P:614-619 by central differences,
    away from the kinks (|l_n|, R, l_t* bounded away from 0 by 1e-3)."""
    rng = np.random.default_rng(13)
    h = 1e-7
    n_checked = 0
    for _ in range(3000):
        d = rng.choice([2, 3])
        v = rng.standard_normal(d)
        n = rng.standard_normal(d)
        n /= np.linalg.norm(n)
        c = rng.uniform(0.0, 2.0)
        ln = v @ n
        vt = v - ln * n
        lt = np.sqrt(vt @ vt + 1e-10)
        R = lt + c * min(ln, 0.0)
        if abs(ln) < 1e-3 or abs(R) < 1e-3:
            continue
        J = np.zeros((d, d))
        for a in range(d):
            e = np.zeros(d)
            e[a] = h
            J[:, a] = (oracle.project(v + e, n, c) - oracle.project(v - e, n, c)) / (2 * h)
        g = rng.standard_normal(d)
        adj = oracle.project_adj(v, n, c, g)
        np.testing.assert_allclose(adj, J.T @ g, atol=1e-6 * max(1.0, np.abs(J.T @ g).max()))
        n_checked += 1
    assert n_checked > 1000


# ---- grid operation, steps D, E --------------------------------------------------
def test_grid_ops_golden():
    cfg = oracle.Config(dim=2, res=64, dt=1e-3, gravity=(0.0, 0.0))
    node = [32, 32]
    for row in _rows("grid_ops.txt"):
        t = row.split()
        kind, m, px, py, dvx, dvy = t[0], *(float(s) for s in t[1:6])
        exp = [float(s) for s in t[6:]]
        if kind == "v":
            vbar, v = oracle.grid_node(cfg, node, m, [px, py])
            np.testing.assert_allclose(v, exp, atol=1e-15)
        elif kind == "dp":
            dp, _ = oracle.grid_node_adj(cfg, node, m, [px, py], [dvx, dvy])
            np.testing.assert_allclose(dp, exp, atol=1e-15)
        else:
            _, dm = oracle.grid_node_adj(cfg, node, m, [px, py], [dvx, dvy])
            assert abs(dm - exp[0]) < 1e-15


def test_grid_node_adjoint_fd():
    """Steps L, D, E composed on band nodes (corners included) vs central differences of the
    node map (m, p) -> v, kinks excluded."""
    rng = np.random.default_rng(14)
    h = 1e-7
    checked = 0
    for _ in range(2000):
        d = int(rng.choice([2, 3]))
        res = 16
        fr = tuple(rng.uniform(0, 1.5, 6))
        cfg = oracle.Config(dim=d, res=res, dt=1e-3, gravity=tuple(rng.standard_normal(3)),
                            bound=3, friction=fr)
        node = rng.choice([0, 1, 2, 7, 13, 14, 15], d)
        m = rng.uniform(0.5, 2.0)
        p = rng.standard_normal(d)
        g = rng.standard_normal(d)

        def f(m_, p_):
            return oracle.grid_node(cfg, node, m_, p_)[1]

        base = f(m, p)
        Jp = np.zeros((d, d))
        for a in range(d):
            e = np.zeros(d)
            e[a] = h
            Jp[:, a] = (f(m, p + e) - f(m, p - e)) / (2 * h)
        Jm = (f(m + h, p) - f(m - h, p)) / (2 * h)
        # skip configurations within 1e-4 of a kink (FD straddles it)
        J2 = np.zeros((d, d))
        for a in range(d):
            e = np.zeros(d)
            e[a] = 0.1 * h
            J2[:, a] = (f(m, p + e) - f(m, p - e)) / (0.2 * h)
        if np.abs(J2 - Jp).max() > 1e-4 * max(1, np.abs(Jp).max()):
            continue
        dp, dm = oracle.grid_node_adj(cfg, node, m, p, g)
        np.testing.assert_allclose(dp, Jp.T @ g, atol=2e-6 * max(1, np.abs(Jp).max()))
        assert abs(dm - Jm @ g) < 2e-6 * max(1, abs(Jm @ g))
        checked += 1
    assert checked > 1000


def test_wall_bands_golden():
    """Hand-derived step L per wall band (golden/walls.txt): pins which wall gets which c and
    normal sign in the oracle's band geometry (R6), the sticky flag per wall, the R < 0 full
    stop, the axis order at corners, and the adjoint (steps L, D, E) on the same nodes."""
    n_rows = 0
    for row in _rows("walls.txt"):
        lhs, rhs = row.split("->")
        t = lhs.split()
        kind, d = t[0], int(t[1])
        fr = tuple(float(s) for s in t[2:8])
        node = [int(s) for s in t[8:8 + d]]
        m = float(t[8 + d])
        p = [float(s) for s in t[9 + d:9 + 2 * d]]
        exp = [float(s) for s in rhs.split()]
        cfg = oracle.Config(dim=d, res=16, dt=1e-3, gravity=(0.0, 0.0, 0.0), bound=3, friction=fr)
        if kind == "fwd":
            _, v = oracle.grid_node(cfg, node, m, p)
            np.testing.assert_allclose(v, exp, atol=1e-8, err_msg=row)
        else:
            g = [float(s) for s in t[9 + 2 * d:9 + 3 * d]]
            dp, dm = oracle.grid_node_adj(cfg, node, m, p, g)
            np.testing.assert_allclose(dp, exp[:d], atol=1e-8, err_msg=row)
            assert abs(dm - exp[d]) < 1e-8, (row, dm)
        n_rows += 1
    assert n_rows >= 20
