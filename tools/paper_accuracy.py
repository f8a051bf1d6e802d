"""The paper's gradient-accuracy cases A1 and A2 (Table II; cases P:223-224) on
the GPU path, in fp32, against their exact values:
  A1 (3D, analytic): a body in free flight, L = CoM_x(T): dL/dx0_p = m_p/M, dL/dv0_p = T dt m_p/M
      for any internal stress and actuation (no wall contact).
  A2 (3D, analytic + wall): a block sliding into the frictionless +x wall (c = 0, g = 0),
      L = CoM_y(T): dL/dv0_{p,y} = T dt m_p/M (step L keeps tangential velocity).
The paper's error metric is undefined (R16); we print the norm-wise relative error of the
dL/dx0 (A1) / dL/dv0 (A2) fields next to the paper's numbers (another GPU, other scenes).
  python tools/paper_accuracy.py > profiles/r01_paper_accuracy.jsonl"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1810_01054_b200 import mpm, scenes  # noqa: E402

PAPER_A1 = {1: 9.80e-8, 10: 4.74e-8, 100: 1.15e-7, 1000: 1.43e-5}
FUSE = int(os.environ.get("MPM_FUSE", "0"))  # 1: the fused G2P2G forward (NEXT N2)
PAPER_A2 = {1000: 2.69e-5}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def a1(T):
    sc = scenes.slab_3d(steps=T, cells=(20, 20, 20), res=64, y0=22)  # 64,000 particles, actuated
    sc.gravity = (0.0, -9.8, 0.0)
    sc.v[..., 0] = 0.2
    sc.v[..., 1] = 0.0
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, checkpoint_every=min(T, 100), fuse_g2p2g=FUSE))
    sim.set_scene(sc)
    sim.forward(T)
    m = sc.mass[0].astype(np.float64)
    M = m.sum()
    seed = np.zeros((sc.n, 3), np.float32)
    seed[:, 0] = (m / M).astype(np.float32)
    sim.backward(seed)
    g = sim.grad()
    ex = np.zeros(3)
    ex[0] = 1.0
    out = {"case": "A1", "fuse_g2p2g": FUSE, "steps": T, "particles": sc.n,
           "rel_err_dx0": rel(g["dx0"], (m / M)[:, None] * ex),
           "rel_err_dv0": rel(g["dv0"], (T * sc.dt * m / M)[:, None] * ex),
           "paper_table2_f32": PAPER_A1[T]}
    sim.close()
    return out


def a2(T):
    res = 64
    sc = scenes.slab_3d(steps=T, cells=(12, 12, 12), res=res, y0=26)
    sc.gravity = (0.0, 0.0, 0.0)
    sc.friction = (0.0,) * 6
    sc.x[..., 0] += np.float32(18.0 / res)  # start 18 cells closer to the +x wall
    sc.v[..., 0] = 1.0   # reaches the wall band within the horizon (6.4 cells)
    sc.v[..., 1] = 0.1
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, checkpoint_every=min(T, 100), fuse_g2p2g=FUSE))
    sim.set_scene(sc)
    sim.forward(T)
    v = sim.get_state(T)[1]
    assert v[:, 0].min() < 0.5, "the block never hit the +x wall (its normal velocity is intact)"
    m = sc.mass[0].astype(np.float64)
    M = m.sum()
    seed = np.zeros((sc.n, 3), np.float32)
    seed[:, 1] = (m / M).astype(np.float32)
    sim.backward(seed)
    g = sim.grad()
    ey = np.array([0.0, 1.0, 0.0])
    out = {"case": "A2", "fuse_g2p2g": FUSE, "steps": T, "particles": sc.n,
           "rel_err_dv0": rel(g["dv0"], (T * sc.dt * m / M)[:, None] * ey),
           "rel_err_dx0": rel(g["dx0"], (m / M)[:, None] * ey),
           "paper_table2_f32": PAPER_A2[T]}
    sim.close()
    return out


if __name__ == "__main__":
    for T in (1, 10, 100, 1000):
        print(json.dumps(a1(T)), flush=True)
    print(json.dumps(a2(1000)), flush=True)
