"""Seeded randomised parity sweep of the whole step (forward Eqs. 3-10, reverse steps A-L)
against the fp64 oracle.  Drawn per case: dimension, grid resolution, block count and shape
(ragged blocks at every size), placement (including the wall bands), per-wall friction,
gravity, actuator count and strength, material (R1 / R21), fused or unfused forward (N2),
checkpoint interval (N2), the mass gradient (N3), running-loss seeds on intermediate states
(N4) and the horizon -- so that combinations the hand-written cases do not name are
exercised too.  Bars as in the other parity tests: state at the field scale 1e-4, gradients
1e-3 norm-wise (R16) and element-wise at the field scale; binning bit-exact at every resident step."""
import os

import numpy as np
import pytest

import oracle
from paper_1810_01054_b200 import mpm, scenes
from tests.helpers import assert_grads, oracle_cfg, oracle_params, oracle_state, rel_err

pytestmark = pytest.mark.gpu

# MPM_SWEEP_CASES / MPM_SWEEP_SEED (default 160 / 0): a longer or different sweep on demand
N_CASES = int(os.environ.get("MPM_SWEEP_CASES", "160"))
SEED0 = int(os.environ.get("MPM_SWEEP_SEED", "0"))
# per-wall friction draws: sticky (c < 0, R6), frictionless, sliding, and the full stop of
# step L (c >= 1 stops a node whose |l_n| exceeds l_t / c: R < 0, H(R) = 0)
FRICTIONS = [-1.0, 0.0, 0.5, 1.0, 2.0]


def _case(i):
    rng = np.random.default_rng(9100 + SEED0 + i)
    d = 2 + i % 2
    res = int(rng.choice([16, 32, 64]))
    n_cells = tuple(int(c) for c in rng.integers(1, 11, d))
    # low corner of the block (cells); margins of one cell below and two above keep every base
    # index in [0, res - 3] while the block may sit inside the wall bands
    lo = tuple(int(rng.integers(1, res - n_cells[a] - 1)) for a in range(d))
    K = int(rng.integers(0, 4))
    T = int(rng.integers(2, 13))
    fric = tuple(float(rng.choice(FRICTIONS)) for _ in range(2 * d)) + (0.0,) * (6 - 2 * d)
    g = tuple(float(v) for v in rng.uniform(-10.0, 10.0, d))
    sc = scenes.tiny(d, seed=9200 + SEED0 + i, res=res, n_cells=n_cells, center=lo, steps=T, K=K,
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
    assert_grads(pairs, ctx=o)


N_BATCH_CASES = int(os.environ.get("MPM_SWEEP_BATCH_CASES", "32"))


def _batch_case(i):
    """B rollouts of the same size in one context (the batch dimension of the launch grid, C5b):
    each its own block placement, velocities, F0, C0, E, actuation, so the rollouts' blocks
    interleave in the block table differently at every step."""
    import dataclasses
    rng = np.random.default_rng(9500 + SEED0 + i)
    d = 2 + i % 2
    B = int(rng.integers(2, 5))
    res = int(rng.choice([16, 32]))
    n_cells = tuple(int(c) for c in rng.integers(1, 7, d))
    K = int(rng.integers(0, 3))
    T = int(rng.integers(2, 9))
    fric = tuple(float(rng.choice(FRICTIONS)) for _ in range(2 * d)) + (0.0,) * (6 - 2 * d)
    g = tuple(float(v) for v in rng.uniform(-10.0, 10.0, d))
    s = float(rng.uniform(0.0, 50.0))
    parts = []
    for r in range(B):
        lo = tuple(int(rng.integers(1, res - n_cells[a] - 1)) for a in range(d))
        parts.append(scenes.tiny(d, seed=9600 + 16 * i + r, res=res, n_cells=n_cells, center=lo, steps=T, K=K,
                                 s=s, gravity=g, friction=fric))
    cat = lambda k: np.concatenate([getattr(p, k) for p in parts], axis=0)
    sc = dataclasses.replace(parts[0], **{k: cat(k) for k in ("x", "v", "F", "C", "mass", "vol", "E", "nu",
                                                                "actuator_id", "act")})
    return sc, T, dict(fuse=int(rng.integers(0, 2)), material=int(i % 4 == 3))


@pytest.mark.parametrize("i", range(N_BATCH_CASES))
def test_random_batch_forward_backward(i):
    sc, T, o = _batch_case(i)
    d, B, n = sc.dim, sc.batch, sc.n
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, material=o["material"], fuse_g2p2g=o["fuse"]))
    sim.set_scene(sc)
    sim.forward(T)
    for t in range(T):  # a1: keys (rollout, block, cell), stable ties, over the whole batch
        xs, orig, key, perm, bs = sim.get_binning(t)
        okey, operm, obs = oracle.bin_particles(d, sc.res, xs.reshape(B, n, d))
        np.testing.assert_array_equal(key, okey)
        np.testing.assert_array_equal(perm, operm)
        np.testing.assert_array_equal(bs, obs)
    x, v, F, Cm = sim.get_state(T)
    rng = np.random.default_rng(9700 + i)
    seeds, trajs, cfg = [], [], oracle_cfg(sc, material=o["material"])
    for r in range(B):
        m, vol, E, nu, aid, act = oracle_params(sc, r)
        traj = oracle.forward(cfg, oracle_state(sc, r), m, vol, E, nu, aid, act[:T], T)
        trajs.append(traj)
        ox, ov, oC, oF = oracle.unpack(traj[T], d)
        sl = slice(r * n, (r + 1) * n)
        vmax = max(np.abs(ov).max(), 1e-6)
        for k, a, b, scale in (("x", x[sl], ox, 1.0), ("v", v[sl], ov, vmax),
                               ("F", F[sl], oF, np.abs(oF).max()), ("C", Cm[sl], oC, 4 * sc.res * vmax)):
            err = np.abs(a - b).max() / scale
            assert err < 1e-4, (r, k, err)
        seeds.append(rng.standard_normal(traj[T].shape))
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    un = [oracle.unpack(w, d) for w in seeds]
    sim.backward(*(f32(np.concatenate([u[q] for u in un])) for q in (0, 1, 3, 2)))  # x, v, F, C
    g = sim.grad()
    for r in range(B):
        m, vol, E, nu, aid, act = oracle_params(sc, r)
        g0, gE, gnu, ga = oracle.backward(cfg, trajs[r], m, vol, E, nu, aid, act[:T], seeds[r])
        gx, gv, gC, gF = oracle.unpack(g0, d)
        sl = slice(r * n, (r + 1) * n)
        pairs = [("dx0", g["dx0"][sl], gx), ("dv0", g["dv0"][sl], gv), ("dF0", g["dF0"][sl], gF),
                 ("dC0", g["dC0"][sl], gC), ("dE", g["dE"][sl], gE), ("dnu", g["dnu"][sl], gnu)]
        if sc.n_act > 0:
            pairs.append(("da", g["da"][r, :T], ga))
        assert_grads(pairs, ctx=(r, o))


N_SLAB_CASES = int(os.environ.get("MPM_SWEEP_SLAB_CASES", "24"))


def _slab_case(i):
    """One body spread along x, split into G x-slabs at particle-balanced block
    boundaries: random slab count, halo width, grid, body extent, drift speed across the
    slab boundaries, gravity, friction and actuators."""
    from paper_1810_01054_b200 import parallel
    rng = np.random.default_rng(9800 + SEED0 + i)
    d = 2 + i % 2
    res = int(rng.choice([32, 64])) if d == 3 else int(rng.choice([64, 128]))
    nbp = res // parallel.block_size(d)
    halo = int(rng.choice([1, 1, 2]))
    G = int(rng.integers(2, min(4, nbp // (2 * halo)) + 1))
    nx = int(rng.integers(res // 2, res - 4))
    n_cells = (nx,) + tuple(int(c) for c in rng.integers(1, 5, d - 1))
    lo = (int(rng.integers(1, res - nx - 1)),) + tuple(int(rng.integers(4, res - 9)) for _ in range(d - 1))
    T = int(rng.integers(2, 11))
    fric = tuple(float(rng.choice(FRICTIONS)) for _ in range(2 * d)) + (0.0,) * (6 - 2 * d)
    g = tuple(float(v) for v in rng.uniform(-10.0, 10.0, d))
    v0 = (float(rng.choice([-1.0, 1.0]) * rng.uniform(0.0, 8.0)),) + (0.0,) * (d - 1)
    sc = scenes.tiny(d, seed=9900 + SEED0 + i, res=res, n_cells=n_cells, center=lo, steps=T,
                     K=int(rng.integers(0, 3)), s=float(rng.uniform(0.0, 50.0)), gravity=g,
                     friction=fric, v0=v0)
    while G > 2:  # every slab owns particles (the ABI requires n_particles >= 1 per context)
        bounds = parallel.slab_partition(sc.x[0], sc.res, d, G, halo)
        if all(len(parallel.slab_members(sc.x[0], sc.res, a, b)) for a, b in bounds):
            break
        G -= 1
    return sc, T, G, halo


@pytest.mark.parametrize("i", range(N_SLAB_CASES))
def test_random_slab_split(i):
    from tests.test_gpu_slab import _check_slab_run
    sc, T, G, halo = _slab_case(i)
    _check_slab_run(sc, T, G, halo, seed=9950 + i)


N_CTRL_CASES = int(os.environ.get("MPM_SWEEP_CTRL_CASES", "16"))


@pytest.mark.parametrize("i", range(N_CTRL_CASES))
def test_random_controller(i):
    """NEXT N1 on random scenes: a_t = tanh(W z_t + b) from the state each step, random
    actuator count, weight scale, bias and target; state, every state/parameter gradient and
    dL/dW, dL/db, dL/dtarget against the controller oracle (oracle/controller.py)."""
    from oracle import controller as ctl
    rng = np.random.default_rng(10100 + SEED0 + i)
    d = 2 + i % 2
    res = int(rng.choice([16, 32]))
    n_cells = tuple(int(c) for c in rng.integers(2, 9, d))
    lo = tuple(int(rng.integers(1, res - n_cells[a] - 1)) for a in range(d))
    K = int(rng.integers(1, 5))
    T = int(rng.integers(2, 16))
    sc = scenes.tiny(d, seed=10200 + SEED0 + i, res=res, n_cells=n_cells, center=lo, steps=T, K=K,
                     s=float(rng.uniform(10.0, 50.0)),
                     friction=tuple(float(rng.choice([0.0, 0.5])) for _ in range(2 * d)) + (0.0,) * (6 - 2 * d))
    nz = ctl.n_obs(d, K)
    W = (rng.standard_normal((K * d, nz)) * rng.uniform(0.05, 1.0)).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, K * d).astype(np.float32)
    target = rng.uniform(0.2, 0.8, d).astype(np.float32)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T))
    sim.set_scene(sc)
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
        assert rel_err(a_, b_) < 1e-3, (k, rel_err(a_, b_))
    og, ogE, ognu, ogW, ogb, ogt, oga = ctl.backward(cfg, traj, m, vol, E, nu, aid, W64, b64, acts, zs, w)
    gx, gv, gC, gF = oracle.unpack(og, d)
    assert_grads([("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF), ("dC0", g["dC0"], gC),
                  ("dE", g["dE"], ogE), ("dnu", g["dnu"], ognu), ("da", g["da"][0, :T], oga),
                  ("dW", gW, ogW), ("db", gb, ogb), ("dtarget", gt, ogt)])
    sim.close()


@pytest.mark.parametrize("i", range(0, 64, 4))
def test_random_scene_graph_replay(i):
    """The sweep's scenes with the step loops replayed as CUDA graphs (mpm_set_graphs): the
    first pass captures (or, for checkpointed runs, falls back to plain launches), the second
    replays; both against the oracle."""
    import torch
    sc, T, o = _case(i)
    d = sc.dim
    stream = torch.cuda.Stream()
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, material=o["material"], fuse_g2p2g=o["fuse"],
                                        checkpoint_every=o["ck"], stream=stream.cuda_stream))
    sim.set_scene(sc)
    sim.set_graphs(True)
    sim.enable_mass_grad(o["mass_grad"])
    cfg = oracle_cfg(sc, material=o["material"])
    m, vol, E, nu, aid, act = oracle_params(sc)
    traj = oracle.forward(cfg, oracle_state(sc), m, vol, E, nu, aid, act[:T], T)
    W = np.zeros(traj.shape)
    W[T] = np.random.default_rng(9400 + i).standard_normal(traj[T].shape)
    g0, gE, gnu, ga, ogm = oracle.backward_ex(cfg, traj, m, vol, E, nu, aid, act[:T], W)
    gx, gv, gC, gF = oracle.unpack(g0, d)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    wx, wv, wC, wF = oracle.unpack(W[T], d)
    for _ in range(2):
        sim.rewind(0)
        sim.forward(T)
        x, v, F, Cm = sim.get_state(T)
        vmax = max(np.abs(ov).max(), 1e-6)
        for k, a, b, scale in (("x", x, ox, 1.0), ("v", v, ov, vmax), ("F", F, oF, np.abs(oF).max()),
                               ("C", Cm, oC, 4 * sc.res * vmax)):
            assert np.abs(a - b).max() / scale < 1e-4, k
        sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
        g = sim.grad()
        pairs = [("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dF0", g["dF0"], gF),
                 ("dC0", g["dC0"], gC), ("dE", g["dE"], gE), ("dnu", g["dnu"], gnu)]
        if sc.n_act > 0:
            pairs.append(("da", g["da"][0, :T], ga))
        if o["mass_grad"]:
            pairs.append(("dm", sim.grad_mass(), ogm))
        assert_grads(pairs, ctx=o)
    sim.close()
