"""Seeded randomised parity sweep of the whole step (forward Eqs. 3-10, reverse steps A-L)
against the fp64 oracle.  Drawn per case: dimension, grid resolution, block count and shape
(ragged blocks at every size), placement (including the wall bands), per-wall friction,
gravity, actuator count and strength, material (R1 / R21), fused or unfused forward (N2),
checkpoint interval (N2), the mass gradient (N3), running-loss seeds on intermediate states
(N4) and the horizon -- so that combinations the hand-written cases do not name are
exercised too.  Bars as in the other parity tests: state at the field scale 1e-4, gradients
1e-3 (norm-wise, R16); binning bit-exact at every resident step."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm, scenes
from tests.helpers import oracle_cfg, oracle_params, oracle_state, rel_err

pytestmark = pytest.mark.gpu

N_CASES = 160


def _case(i):
    rng = np.random.default_rng(9100 + i)
    d = 2 + i % 2
    res = int(rng.choice([16, 32, 64]))
    n_cells = tuple(int(c) for c in rng.integers(1, 11, d))
    # low corner of the block (cells); margins of one cell below and two above keep every base
    # index in [0, res - 3] while the block may sit inside the wall bands
    lo = tuple(int(rng.integers(1, res - n_cells[a] - 1)) for a in range(d))
    K = int(rng.integers(0, 4))
    T = int(rng.integers(2, 13))
    fric = tuple(float(rng.choice([0.0, 0.5])) for _ in range(2 * d)) + (0.0,) * (6 - 2 * d)
    g = tuple(float(v) for v in rng.uniform(-10.0, 10.0, d))
    sc = scenes.tiny(d, seed=9200 + i, res=res, n_cells=n_cells, center=lo, steps=T, K=K,
                     s=float(rng.uniform(0.0, 50.0)), gravity=g, friction=fric)
    opts = dict(material=int(i % 4 == 3), fuse=int(rng.integers(0, 2)),
                ck=int(rng.choice([0, 0, 2, 3, 5])), mass_grad=bool(rng.integers(0, 2)),
                seeds=bool(rng.integers(0, 2)))
    if opts["ck"] > T:  # the ABI requires checkpoint_every <= max_steps
        opts["ck"] = 0
    return sc, T, opts


@pytest.mark.parametrize("i", range(N_CASES))
def test_random_scene_forward_backward(i):
    sc, T, o = _case(i)
    d = sc.dim
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, material=o["material"], fuse_g2p2g=o["fuse"],
                                        checkpoint_every=o["ck"]))
    sim.set_scene(sc)
    sim.enable_mass_grad(o["mass_grad"])
    sim.forward(T)
    if not o["ck"]:  # a1: bit-exact binning of every step (checkpointed runs keep one segment)
        for t in range(T):
            xs, orig, key, perm, bs = sim.get_binning(t)
            okey, operm, obs = oracle.bin_particles(d, sc.res, xs.reshape(1, -1, d))
            np.testing.assert_array_equal(key, okey)
            np.testing.assert_array_equal(perm, operm)
            np.testing.assert_array_equal(bs, obs)
    cfg = oracle_cfg(sc, material=o["material"])
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    x, v, F, Cm = sim.get_state(T)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    vmax = max(np.abs(ov).max(), 1e-6)
    for k, a, b, scale in (("x", x, ox, 1.0), ("v", v, ov, vmax), ("F", F, oF, np.abs(oF).max()),
                           ("C", Cm, oC, 4 * sc.res * vmax)):
        err = np.abs(a - b).max() / scale
        assert err < 1e-4, (k, err)
    rng = np.random.default_rng(9300 + i)
    W = np.zeros(traj.shape)
    W[T] = rng.standard_normal(traj[T].shape)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    if o["seeds"]:  # N4: a running loss on a random subset of the intermediate states
        for t in np.flatnonzero(rng.random(T) < 0.4):
            W[t] = rng.standard_normal(traj[t].shape)
            wx, wv, wC, wF = oracle.unpack(W[t], d)
            sim.add_seed(int(t), f32(wx), f32(wv), f32(wF), f32(wC))
    wx, wv, wC, wF = oracle.unpack(W[T], d)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    g0, gE, gnu, ga, ogm = oracle.backward_ex(cfg, traj, m, vol, E, nu, aid, act[:T], W)
    gx, gv, gC, gF = oracle.unpack(g0, d)
    pairs = [("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF),
             ("dC0", g["dC0"], gC), ("dE", g["dE"], gE), ("dnu", g["dnu"], gnu)]
    if sc.n_act > 0:
        pairs.append(("da", g["da"][0, :T], ga))
    if o["mass_grad"]:
        pairs.append(("dm", sim.grad_mass(), ogm))
    for k, a, b in pairs:
        assert rel_err(a, b) < 1e-3, (k, rel_err(a, b), o)
