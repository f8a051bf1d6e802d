"""Parity margins: norm-wise relative error (reading R16) and element-wise error at the field
scale (tests/helpers.elem_err) of the CUDA path vs the fp64 oracle, per field, for the BASELINE configs C1-C3 and a C5b-style batch; prints one JSON line per case.
Run on a GPU box:  python tools/parity_report.py > profiles/parity_margins.jsonl"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure; this is a report tool, not the product)
from paper_1810_01054_b200 import mpm, scenes  # noqa: E402
from tests.helpers import elem_err, oracle_cfg, rel_err, wall_scenes  # noqa: E402


def case(name, sc, T, r=0, **cfgkw):
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, **cfgkw))
    sim.set_scene(sc)
    sim.enable_mass_grad(True)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    cfg = oracle_cfg(sc, material=cfgkw.get("material", 0))
    st = oracle.pack(sc.x[r], sc.v[r], sc.C[r], sc.F[r])
    prm = [a[r].astype(np.float64) for a in (sc.mass, sc.vol, sc.E, sc.nu)]
    aid, act = sc.actuator_id[r], sc.act[r].astype(np.float64)[:T]
    t0 = time.time()
    traj = oracle.forward(cfg, st, *prm, aid, act, T)
    ox, ov, oC, oF = oracle.unpack(traj[T], sc.dim)
    sl = slice(r * sc.n, (r + 1) * sc.n)
    out = {"case": name, "steps": T, "particles": sc.n,
           "state": {k: rel_err(a[sl], b) for k, a, b in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC))}}
    rng = np.random.default_rng(1)
    S = oracle.S_of(sc.dim)
    w = rng.standard_normal((sc.batch, sc.n, S))
    wx, wv, wC, wF = oracle.unpack(w.reshape(-1, S), sc.dim)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    gm = sim.grad_mass()
    seeds = np.zeros_like(traj)
    seeds[T] = w[r]
    g0, gE, gnu, ga, ogm = oracle.backward_ex(cfg, traj, *prm, aid, act, seeds)
    gx, gv, gC, gF = oracle.unpack(g0, sc.dim)
    gp = (
        ("dx0", g["dx0"][sl], gx), ("dv0", g["dv0"][sl], gv), ("dF0", g["dF0"][sl], gF),
        ("dC0", g["dC0"][sl], gC), ("dE", g["dE"][sl], gE), ("dnu", g["dnu"][sl], gnu),
        ("da", g["da"][r, :T], ga), ("dm", gm[sl], ogm))
    out["grad"] = {k: rel_err(a, b) for k, a, b in gp}
    out["grad_elem"] = {k: elem_err(a, b) for k, a, b in gp}
    out["oracle_s"] = round(time.time() - t0, 1)
    sim.close()
    print(json.dumps(out), flush=True)


def controller_case(name, sc, T, scale=0.2):
    from oracle import controller as ctl
    K, d = sc.n_act, sc.dim
    rng = np.random.default_rng(7)
    W = (rng.standard_normal((K * d, ctl.n_obs(d, K))) * scale).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, K * d).astype(np.float32)
    target = rng.uniform(0.2, 0.8, d).astype(np.float32)
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T))
    sim.set_scene(sc)
    sim.set_controller(W, b, target)
    sim.forward(T)
    x, v, F, Cm = sim.get_state(T)
    cfg = oracle_cfg(sc)
    m, vol, E, nu = (a[0].astype(np.float64) for a in (sc.mass, sc.vol, sc.E, sc.nu))
    t0 = time.time()
    traj, acts, zs = ctl.forward(cfg, oracle.pack(sc.x[0], sc.v[0], sc.C[0], sc.F[0]), m, vol, E, nu,
                                 sc.actuator_id[0], W.astype(np.float64), b.astype(np.float64),
                                 target.astype(np.float64), T)
    ox, ov, oC, oF = oracle.unpack(traj[T], d)
    w = np.random.default_rng(1).standard_normal(traj[T].shape)
    wx, wv, wC, wF = oracle.unpack(w, d)
    f32 = lambda a: np.ascontiguousarray(a, np.float32)
    sim.backward(f32(wx), f32(wv), f32(wF), f32(wC))
    g = sim.grad()
    gW, gb, gt = sim.grad_controller()
    og, _, _, ogW, ogb, ogt, _ = ctl.backward(cfg, traj, m, vol, E, nu, sc.actuator_id[0], W.astype(np.float64),
                                             b.astype(np.float64), acts, zs, w)
    gx, gv, gC, gF = oracle.unpack(og, d)
    gp = (("dx0", g["dx0"], gx), ("dv0", g["dv0"], gv), ("dW", gW, ogW), ("db", gb, ogb), ("dtarget", gt, ogt))
    out = {"case": name, "steps": T, "particles": sc.n,
           "state": {k: rel_err(a_, b_) for k, a_, b_ in (("x", x, ox), ("v", v, ov), ("F", F, oF), ("C", Cm, oC))},
           "grad": {k: rel_err(a_, b_) for k, a_, b_ in gp},
           "grad_elem": {k: elem_err(a_, b_) for k, a_, b_ in gp},
           "oracle_s": round(time.time() - t0, 1)}
    sim.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    case("C1 configs[0] 2D block", scenes.block_2d(steps=50, perturb=True), 50)
    case("C2 configs[1] 2D walker", scenes.walker_2d(steps=100), 100)
    case("C2 configs[1] 2D walker, 500 steps", scenes.walker_2d(steps=500), 500)
    case("C3 configs[2] 3D quadruped", scenes.quadruped_3d(steps=100), 100)
    case("C3 configs[2] 3D quadruped, 200 steps", scenes.quadruped_3d(steps=200), 200)
    case("C5b-style batch (rollout 2 of 3)", scenes.quadruped_3d(batch=3, steps=50, e_scale=True), 50, r=2)
    case("C3 fixed-corotated (N3, R21)", scenes.quadruped_3d(steps=100), 100, material=1)
    case("C2 fixed-corotated (N3, R21)", scenes.walker_2d(steps=200), 200, material=1)
    case("C3 checkpoint_every=16 (N2)", scenes.quadruped_3d(steps=100), 100, checkpoint_every=16)
    case("C1 fused G2P2G (N2)", scenes.block_2d(steps=50, perturb=True), 50, fuse_g2p2g=1)
    case("C2 fused G2P2G (N2), 500 steps", scenes.walker_2d(steps=500), 500, fuse_g2p2g=1)
    case("C3 fused G2P2G (N2), 200 steps", scenes.quadruped_3d(steps=200), 200, fuse_g2p2g=1)
    case("C3 fused G2P2G + checkpoint_every=16 + fixed-corotated", scenes.quadruped_3d(steps=100), 100,
         fuse_g2p2g=1, checkpoint_every=16, material=1)
    controller_case("C2 closed-loop controller (N1), 200 steps", scenes.walker_2d(steps=200), 200)
    controller_case("C3 closed-loop controller (N1), 60 steps", scenes.quadruped_3d(steps=60), 60, 0.1)
    # step L with every wall kind: sticky (c < 0) and full-stop (c >= 1, R < 0 -> H(R) = 0) walls
    for d in (2, 3):
        for name, sc in wall_scenes(d, 60):
            case(name, sc, 60)
