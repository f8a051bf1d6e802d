"""GPU parity of step L with every kind of wall (DESIGN R6-R8): sticky walls (c < 0),
high-friction walls whose projection stops the node (c >= 1: R = l_t + c l_n < 0, so l_t* = 0
and H(R) = 0 in the adjoint) and sliding walls (0 < c < 1), on
blocks driven into the low corner and into the high corner of the domain, against the fp64
oracle: state at the field scale and every gradient family element-wise (tests/helpers
assert_grads), unfused and fused (G2P2G) forward."""
import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm
from tests.helpers import assert_grads, oracle_cfg, oracle_params, oracle_state, wall_scenes

pytestmark = pytest.mark.gpu

T = 60
CASES = [(d, i, fuse) for d in (2, 3) for i in (0, 1) for fuse in (0, 1)]


@pytest.mark.parametrize("d,i,fuse", CASES)
def test_walls_forward_backward(d, i, fuse):
    name, sc = wall_scenes(d, T)[i]
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, fuse_g2p2g=fuse))
    sim.set_scene(sc)
    sim.enable_mass_grad(True)
    sim.forward(T)
    cfg = oracle_cfg(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    x, v, F, Cm = sim.get_state(T)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    v0max = np.abs(sc.v[0]).max()
    for k, a, b, scale in (("x", x, ox, 1.0), ("v", v, ov, v0max), ("F", F, oF, np.abs(oF).max()),
                           ("C", Cm, oC, 4 * sc.res * v0max)):
        err = np.abs(a - b).max() / scale
        assert err < 1e-4, (name, k, err)
    # the walls act: the block has been (nearly) stopped from |v0| = 1.5
    assert np.abs(ov.mean(0)).max() < 0.5 * v0max, ov.mean(0)
    rng = np.random.default_rng(600 + 10 * d + i)
    W = np.zeros(traj.shape)
    W[T] = rng.standard_normal(traj[T].shape)
    wx, wv, wC, wF = oracle.unpack(W[T], d)
    f32 = lambda q: np.ascontiguousarray(q, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    g0, gE, gnu, ga, ogm = oracle.backward_ex(cfg, traj, m, vol, E, nu, aid, act[:T], W)
    gx, gv, gC, gF = oracle.unpack(g0, d)
    assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF), ("dC0", g["dC0"], gC),
                  ("dE", g["dE"], gE), ("dnu", g["dnu"], gnu), ("da", g["da"][0, :T], ga),
                  ("dm", sim.grad_mass(), ogm)], ctx=name)
    sim.close()
