"""CUDA-graph replay of the step loops (include/mpm.h mpm_set_graphs): a captured forward /
backward loop replayed over new initial states, split forward calls, running-loss seeds and
the mass gradient must give what plain launches give -- checked against the fp64 oracle at
the parity bars (state 1e-4 at the field scale, gradients 1e-3) -- and count the same
launches."""
import numpy as np
import pytest
import torch

import oracle
from paper_1810_01054_b200 import mpm, scenes
from tests.helpers import assert_grads, oracle_cfg, oracle_params, oracle_state, rel_err, run_oracle

pytestmark = pytest.mark.gpu


def _check(sim, sc, T, seed, W=None):
    d = sc.dim
    cfg = oracle_cfg(sc)
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    x, v, F, Cm = sim.get_state(T)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    vmax = max(np.abs(ov).max(), 1e-6)
    for k, a, b, scale in (("x", x, ox, 1.0), ("v", v, ov, vmax), ("F", F, oF, np.abs(oF).max()),
                           ("C", Cm, oC, 4 * sc.res * vmax)):
        assert np.abs(a - b).max() / scale < 1e-4, k
    if W is None:
        W = np.zeros(traj.shape)
        W[T] = np.random.default_rng(seed).standard_normal(traj[T].shape)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    wx, wv, wC, wF = oracle.unpack(W[T], d)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    g0, gE, gnu, ga, gm = oracle.backward_ex(cfg, traj, m, vol, E, nu, aid, act[:T], W)
    gx, gv, gC, gF = oracle.unpack(g0, d)
    pairs = [("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF), ("dC0", g["dC0"], gC),
             ("dE", g["dE"], gE), ("dnu", g["dnu"], gnu), ("da", g["da"][0, :T], ga)]
    assert_grads(pairs)
    return traj, gm


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("fuse", [0, 1])
def test_graph_replay_over_new_states(d, fuse):
    T = 9
    stream = torch.cuda.Stream()
    sc0 = scenes.tiny(d, seed=300, res=32, n_cells=(5,) * d, steps=T, K=2, s=30.0)
    sim = mpm.MPM(mpm.Config.from_scene(sc0, max_steps=T, fuse_g2p2g=fuse, stream=stream.cuda_stream))
    sim.set_graphs(True)
    counts = []
    for rep in range(3):  # capture on the first pass, replay on the others (new x, v, F, C, E, a)
        sc = scenes.tiny(d, seed=300 + rep, res=32, n_cells=(5,) * d, steps=T, K=2, s=30.0)
        sim.set_scene(sc)
        n0 = sim.launch_count()
        sim.forward(4)  # split calls: graphs keyed by (start, length)
        sim.forward(T - 4)
        n1 = sim.launch_count()
        _check(sim, sc, T, 310 + rep)
        counts.append(n1 - n0)
    assert counts[0] == counts[1] == counts[2]
    plain = mpm.MPM(mpm.Config.from_scene(sc0, max_steps=T, fuse_g2p2g=fuse, stream=stream.cuda_stream))
    plain.set_scene(sc0)
    n0 = plain.launch_count()
    plain.forward(4)
    plain.forward(T - 4)
    assert plain.launch_count() - n0 == counts[0]  # a replay counts the kernels it launches
    sim.close()
    plain.close()


def test_graphs_follow_seeds_and_mass_gradient():
    """A new running-loss seed step and the mass-gradient switch change what the backward loop
    launches: the captured loops are dropped and recaptured."""
    d, T = 3, 8
    stream = torch.cuda.Stream()
    sc = scenes.tiny(d, seed=320, res=32, n_cells=(4,) * d, steps=T, K=2, s=30.0)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, fuse_g2p2g=1, stream=stream.cuda_stream))
    sim.set_graphs(True)
    sim.set_scene(sc)
    sim.forward(T)
    _check(sim, sc, T, 321)  # captures forward and backward
    _, traj = run_oracle(sc, steps=T)
    rng = np.random.default_rng(322)
    W = np.zeros(traj.shape)
    W[T] = rng.standard_normal(traj[T].shape)
    W[3] = rng.standard_normal(traj[3].shape)
    wx, wv, wC, wF = oracle.unpack(W[3], d)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.add_seed(3, f32(wx), f32(wv), f32(wF), f32(wC))
    sim.enable_mass_grad(True)
    sim.rewind(0)
    sim.forward(T)
    _, gm = _check(sim, sc, T, 323, W=W)
    assert_grads([("dm", sim.grad_mass(), gm)])
    sim.rewind(0)  # replay of the recaptured loops
    sim.forward(T)
    _, gm = _check(sim, sc, T, 324, W=W)
    assert_grads([("dm", sim.grad_mass(), gm)])
    sim.close()


def test_graphs_need_a_stream():
    sc = scenes.tiny(2, seed=330, res=16, steps=2, K=0)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=2))
    with pytest.raises(mpm.MPMError):
        sim.set_graphs(True)
    sim.close()


@pytest.mark.parametrize("T", [7, 10])
def test_graph_replay_actuation_change_and_odd_tape(T):
    """Replays after mpm_set_actuation changed the actuation (the graph reads the buffer, so the
    new values must take effect) and over an odd tape length (the backward loop's adjoint
    ping-pong ends on the other buffer): both against the oracle."""
    d = 3
    stream = torch.cuda.Stream()
    sc = scenes.tiny(d, seed=340, res=32, n_cells=(5,) * d, steps=T, K=2, s=60.0)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, fuse_g2p2g=1, stream=stream.cuda_stream))
    sim.set_graphs(True)
    sim.set_scene(sc)
    for rep in range(3):
        if rep:  # new actuation only, same particles: the captured loops are replayed
            sc.act[:] = np.random.default_rng(341 + rep).standard_normal(sc.act.shape).astype(np.float32)
            a = np.zeros((1, T, sc.n_act, d), np.float32)
            a[0] = sc.act[0, :T]
            sim.set_actuation(a)
            sim.rewind(0)
        n0 = sim.launch_count()
        sim.forward(T)
        assert sim.launch_count() > n0
        _check(sim, sc, T, 350 + rep)
    sim.close()


def test_graph_replay_with_controller():
    """Closed-loop controller (N1) inside captured loops: k_ctrl_observe resets its own group
    sums and counter, and the backward's controller adjoint runs per step; replays over new
    initial states against the controller oracle, dL/dW, dL/db, dL/dtarget included."""
    from oracle import controller as ctl
    d, T, K = 2, 12, 3
    stream = torch.cuda.Stream()
    rng = np.random.default_rng(360)
    nz = ctl.n_obs(d, K)
    W = (0.3 * rng.standard_normal((K * d, nz))).astype(np.float32)
    b = rng.uniform(-0.3, 0.3, K * d).astype(np.float32)
    target = np.array([0.6, 0.4], np.float32)
    sim = None
    for rep in range(3):
        sc = scenes.tiny(d, seed=361 + rep, res=32, n_cells=(6, 5), steps=T, K=K, s=30.0)
        if sim is None:
            sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, stream=stream.cuda_stream))
            sim.set_graphs(True)
        sim.set_scene(sc)
        if rep == 0:  # set_controller drops captured loops; later reps replay them
            sim.set_controller(W, b, target)
        sim.forward(T)
        x, v, F, Cm = sim.get_state(T)
        w = rng.standard_normal((sc.n, oracle.S_of(d)))
        wx, wv, wC, wF = oracle.unpack(w, d)
        f32 = lambda a: np.ascontiguousarray(a, np.float32)
        sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
        g = sim.grad()
        gW, gb, gt = sim.grad_controller()
        cfg = oracle_cfg(sc)
        m, vol, E, nu, aid, _ = oracle_params(sc)
        W64, b64, t64 = W.astype(np.float64), b.astype(np.float64), target.astype(np.float64)
        traj, acts, zs = ctl.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, W64, b64, t64, T)
        ox, ov, oC, oF = oracle.unpack(traj[T], d)
        for k, a_, b_ in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC)):
            assert rel_err(a_, b_) < 1e-3, (rep, k)
        og, ogE, ognu, ogW, ogb, ogt, oga = ctl.backward(cfg, traj, m, vol, E, nu, aid, W64, b64, acts, zs, w)
        gx, gv, gC, gF = oracle.unpack(og, d)
        assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF), ("dC0", g["dC0"], gC),
                      ("dE", g["dE"], ogE), ("da", g["da"][0, :T], oga), ("dW", gW, ogW), ("db", gb, ogb),
                      ("dtarget", gt, ogt)], ctx=rep)
    sim.close()
