"""configs[4] slab part (C5a: 256^3 grid, 8,355,840 particles) at full size, in the launch
configuration bench.py times at N = 1 (one whole-domain slab), and split into two x-slabs
with window sums (the N = 2 decomposition, emulated on one GPU): bit-exact binning, grid
mass / momentum, sampled one-step states vs the oracle, and the exact CoM gradient."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm, parallel, scenes
from tests.helpers import oracle_cfg, rel_err

pytestmark = pytest.mark.gpu

T = 8


@pytest.fixture(scope="module")
def c5a():
    sc = scenes.slab_c5a(steps=T)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T))
    sim.set_slab(0, sc.res, 1)  # bench.py's N = 1 configuration
    sim.set_scene(sc)
    sim.forward(T)
    return sc, sim


def test_c5a_size(c5a):
    sc, _ = c5a
    assert sc.n == 8_355_840 and sc.res == 256


def test_c5a_binning_bit_exact(c5a):
    sc, sim = c5a
    for t in (0, T - 1):
        x, orig, key, perm, bs = sim.get_binning(t)
        okey, operm, obs = oracle.bin_particles(3, sc.res, x.reshape(1, sc.n, 3))
        np.testing.assert_array_equal(key, okey)
        np.testing.assert_array_equal(perm, operm)
        np.testing.assert_array_equal(bs, obs)


def test_c5a_grid_mass_momentum(c5a):
    sc, sim = c5a
    m, vbar = sim.get_grid(T - 1)
    x, v, F, Cm = sim.get_state(T - 1)
    mp = sc.mass[0].astype(np.float64)
    assert abs(m.sum(dtype=np.float64) - mp.sum()) < 1e-5 * mp.sum()
    g = np.array(sc.gravity)
    p = (m[0, :, None].astype(np.float64) * (vbar[0].astype(np.float64) - sc.dt * g))
    np.testing.assert_allclose(p.sum(0), (mp[:, None] * v.astype(np.float64)).sum(0), rtol=1e-4,
                               atol=1e-6 * mp.sum())


def test_c5a_sampled_particles_one_step(c5a):
    """8 sampled particles: GPU state at t+1 vs the oracle stepping each one's 7^3-cell
    neighbourhood from the GPU's state at t (field-scale errors, R16): 1e-5."""
    sc, sim = c5a
    rng = np.random.default_rng(5)
    t = T - 2
    x, v, F, Cm = sim.get_state(t)
    x1, v1, F1, C1 = sim.get_state(t + 1)
    act_t = sc.act[0][t:t + 1].astype(np.float64)
    cell = np.floor(x * sc.res - 0.5)
    for idx in rng.choice(sc.n, 8, replace=False):
        sub = np.nonzero(np.all(np.abs(cell - cell[idx]) <= 3, axis=1))[0]
        cfg = oracle_cfg(sc)
        st = oracle.pack(x[sub], v[sub], Cm[sub], F[sub])
        prm = [a[0][sub].astype(np.float64) for a in (sc.mass, sc.vol, sc.E, sc.nu)]
        traj = oracle.forward(cfg, st, *prm, sc.actuator_id[0][sub], act_t, 1)
        me = int(np.nonzero(sub == idx)[0][0])
        ox, ov, oC, oF = oracle.unpack(traj[1], 3)
        vmax = max(np.abs(v[sub]).max(), np.abs(ov).max())
        for a, b, scale in ((x1[idx], ox[me], 1.0), (v1[idx], ov[me], vmax),
                            (C1[idx], oC[me], 4 * sc.res * vmax), (F1[idx], oF[me], np.abs(oF).max())):
            assert np.abs(a - b).max() < 1e-5 * scale, (idx, a, b, scale)


def _com_check(sc, g):
    m = sc.mass[0].astype(np.float64)
    M = m.sum()
    ex = np.array([1.0, 0.0, 0.0])
    assert rel_err(g["dx0"], (m / M)[:, None] * ex) < 1e-4
    assert rel_err(g["dv0"], (T * sc.dt * m / M)[:, None] * ex) < 1e-4
    assert np.abs(g["da"]).max() < 1e-6


def test_c5a_com_gradient_closed_form(c5a):
    sc, sim = c5a
    m = sc.mass[0].astype(np.float64)
    seed = np.zeros((sc.n, 3), np.float32)
    seed[:, 0] = m / m.sum()
    sim.backward(seed)
    _com_check(sc, sim.grad())


@pytest.mark.parametrize("fuse", [0, 1])
def test_c5a_two_slabs_full_size(c5a, fuse):
    """The N = 2 decomposition at full size: two x-slabs (count-balanced) with window sums
    give the single-context state and the exact CoM gradient (fuse = 1: the fused forward
    bench.py runs at N > 1, windows of grid t+1 summed between two G2P2G launches)."""
    sc, ref = c5a
    bounds = parallel.slab_partition(sc.x[0], sc.res, 3, 2)
    sims, idxs = [], []
    for lo, hi in bounds:
        s2, idx = parallel.shard_slab(sc, lo, hi)
        s = mpm.MPM(mpm.Config.from_scene(s2, max_steps=T, fuse_g2p2g=fuse))
        s.set_slab(lo, hi, 1)
        s.set_scene(s2)
        sims.append(s)
        idxs.append(idx)
    mpm.group_forward(sims, T)
    xr = ref.get_state(T)[0]
    x = np.empty_like(xr)
    for s, idx in zip(sims, idxs):
        x[idx] = s.get_state(T)[0]
    assert rel_err(x, xr) < (1e-5 if fuse else 1e-6)  # fused: fp32 summation order
    m = sc.mass[0].astype(np.float64)
    M = m.sum()
    seeds = [np.ascontiguousarray(np.stack([m[i] / M, 0 * m[i], 0 * m[i]], 1), np.float32) for i in idxs]
    mpm.group_backward(sims, seeds)
    g = {k: np.empty((sc.n, 3)) for k in ("dx0", "dv0")}
    da = None
    for s, idx in zip(sims, idxs):
        gi = s.grad()
        for k in ("dx0", "dv0"):
            g[k][idx] = gi[k]
        da = gi["da"]  # the shared actuation gradient: the same sum on every slab
    g["da"] = da
    _com_check(sc, g)
    for s in sims:
        s.close()


def test_c5a_fused_forward_full_size(c5a):
    """NEXT N2 at full size: the fused G2P2G forward (bench.py's N = 1 configuration: one
    whole-domain slab, no neighbours) gives the unfused state and the exact CoM gradient."""
    sc, ref = c5a
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, fuse_g2p2g=1))
    sim.set_slab(0, sc.res, 1)
    sim.set_scene(sc)
    sim.set_profiling(True)
    sim.forward(T)
    assert sim.profile()["g2p2g"][1] == T
    for a, b in zip(sim.get_state(T), ref.get_state(T)):
        assert rel_err(a, b) < 1e-5
    m = sc.mass[0].astype(np.float64)
    seed = np.zeros((sc.n, 3), np.float32)
    seed[:, 0] = m / m.sum()
    sim.backward(seed)
    _com_check(sc, sim.grad())
    sim.close()
