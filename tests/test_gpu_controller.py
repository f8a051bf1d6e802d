"""NEXT N1 on the GPU: the closed-loop controller a_t = tanh(W z_t + b) embedded in the
forward step, and its adjoint in the backward, against the controller oracle
(oracle/controller.py, pinned by FD in tests/test_oracle_controller.py)."""
import numpy as np
import pytest

import oracle
from oracle import controller as ctl
from paper_1810_01054_b200 import mpm, scenes
from tests.helpers import assert_grads, oracle_cfg, oracle_params, oracle_state, rel_err

pytestmark = pytest.mark.gpu


def _run(sc, T, W, b, target, seed=3):
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T))
    sim.set_scene(sc)
    sim.set_controller(W, b, target)
    sim.forward(T)
    st = sim.get_state(T)
    rng = np.random.default_rng(seed)
    S = oracle.S_of(sc.dim)
    w = rng.standard_normal((sc.batch * sc.n, S))
    wx, wv, wC, wF = oracle.unpack(w, sc.dim)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    return sim, st, w, sim.grad(), sim.grad_controller()


def _params(sc, scale, seed):
    K, d = sc.n_act, sc.dim
    nz = ctl.n_obs(d, K)
    rng = np.random.default_rng(seed)
    W = (rng.standard_normal((K * d, nz)) * scale).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, K * d).astype(np.float32)
    target = rng.uniform(0.2, 0.8, d).astype(np.float32)
    return W, b, target


@pytest.mark.parametrize("name,T,scale", [("tiny2", 40, 0.5), ("tiny3", 30, 0.5), ("C2", 100, 0.2),
                                          ("C3", 50, 0.1)])
def test_controller_state_and_gradients_vs_oracle(name, T, scale):
    if name == "tiny2":
        sc = scenes.tiny(2, seed=41, res=32, n_cells=(8, 8), steps=T, K=3, s=40.0)
    elif name == "tiny3":
        sc = scenes.tiny(3, seed=42, res=32, n_cells=(6, 6, 6), steps=T, K=3, s=40.0)
    else:
        sc = scenes.CONFIGS[name](steps=T)
    W, b, target = _params(sc, scale, 7)
    sim, (x, v, F, Cm), w, g, (gW, gb, gt) = _run(sc, T, W, b, target)
    cfg = oracle_cfg(sc)
    m, vol, E, nu, aid, _ = oracle_params(sc)
    traj, acts, zs = ctl.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, W.astype(np.float64),
                                 b.astype(np.float64), target.astype(np.float64), T)
    ox, ov, oC, oF = oracle.unpack(traj[T], sc.dim)
    for k, a_, b_ in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC)):
        assert rel_err(a_, b_) < 1e-3, (k, rel_err(a_, b_))
    og, ogE, ognu, ogW, ogb, ogt, oga = ctl.backward(cfg, traj, m, vol, E, nu, aid, W.astype(np.float64),
                                                     b.astype(np.float64), acts, zs, w)
    gx, gv, gC, gF = oracle.unpack(og, sc.dim)
    assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF), ("dC0", g["dC0"], gC),
                  ("dE", g["dE"], ogE), ("dnu", g["dnu"], ognu), ("da", g["da"][0, :T], oga),
                  ("dW", gW, ogW), ("db", gb, ogb), ("dtarget", gt, ogt)])
    sim.close()


def test_controller_batch_rollouts_share_parameters():
    """Two rollouts with one controller: dL/dW is the sum of the per-rollout gradients."""
    T = 20
    sc = scenes.quadruped_3d(batch=2, steps=T, e_scale=True)
    W, b, target = _params(sc, 0.1, 9)
    sim, st, w, g, (gW, gb, gt) = _run(sc, T, W, b, target, seed=4)
    cfg = oracle_cfg(sc)
    tot = [np.zeros_like(gW, dtype=np.float64), np.zeros_like(gb, dtype=np.float64)]
    for r in range(2):
        m, vol, E, nu, aid, _ = oracle_params(sc, r)
        traj, acts, zs = ctl.forward(cfg, oracle_state(sc, r), m, vol, E, nu, aid, W.astype(np.float64),
                                     b.astype(np.float64), target.astype(np.float64), T)
        res = ctl.backward(cfg, traj, m, vol, E, nu, aid, W.astype(np.float64), b.astype(np.float64), acts, zs,
                           w[r * sc.n:(r + 1) * sc.n])
        tot[0] += res[3]
        tot[1] += res[4]
        sl = slice(r * sc.n, (r + 1) * sc.n)
        gx = oracle.unpack(res[0], sc.dim)[0]
        assert_grads([("dx0", g["dx0"][sl], gx)], ctx=r)
    assert_grads([("dW", gW, tot[0]), ("db", gb, tot[1])])


def test_controller_errors_and_off_switch():
    sc = scenes.tiny(2, seed=43, res=32, n_cells=(4, 4), steps=4, K=2)
    cfg = mpm.Config.from_scene(sc, max_steps=4)
    s = mpm.MPM(cfg)
    W, b, target = _params(sc, 0.1, 1)
    with pytest.raises(mpm.MPMError) as e:
        s.set_controller(W, b, target)  # before set_state
    assert e.value.status == "MPM_ERR_CALL_ORDER"
    s.set_scene(sc)
    s.forward(2)
    s.backward(np.ones((sc.n, 2), np.float32))
    with pytest.raises(mpm.MPMError) as e:
        s.grad_controller()  # backward ran open-loop
    assert e.value.status == "MPM_ERR_CALL_ORDER"
    # an empty actuator group is an error
    sc2 = scenes.tiny(2, seed=44, res=32, n_cells=(4, 4), steps=4, K=2)
    sc2.actuator_id[:] = np.where(sc2.actuator_id == 1, 0, sc2.actuator_id)
    t = mpm.MPM(mpm.Config.from_scene(sc2, max_steps=4))
    t.set_scene(sc2)
    with pytest.raises(mpm.MPMError) as e:
        t.set_controller(W, b, target)
    assert e.value.status == "MPM_ERR_INVALID_ARG"
    # W = None switches the controller off: the open-loop actuation is used again
    u = mpm.MPM(mpm.Config.from_scene(sc, max_steps=4))
    u.set_scene(sc)
    u.set_controller(W, b, target)
    u.set_controller(None)
    u.forward(4)
    v = mpm.MPM(mpm.Config.from_scene(sc, max_steps=4))
    v.set_scene(sc)
    v.forward(4)
    np.testing.assert_allclose(u.get_state(4)[0], v.get_state(4)[0], rtol=0, atol=1e-6)
