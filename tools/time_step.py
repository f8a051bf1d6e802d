"""Per-kernel device time of the C4 forward + backward step (CUDA events around every
launch inside libmpm).  Usage: python tools/time_step.py [steps] [lib_path]
(MPM_FUSE=1 in the environment: the fused G2P2G forward, NEXT N2; MPM_SCENE=c1|c2|c3 times a
small BASELINE config over K steps instead of C4)"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1810_01054_b200 import mpm, scenes  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    if len(sys.argv) > 2:
        mpm.LIB_PATH = sys.argv[2]
    make = {"c4": scenes.slab_3d, "c1": scenes.block_2d, "c2": scenes.walker_2d,
            "c3": scenes.quadruped_3d}[os.environ.get("MPM_SCENE", "c4")]
    sc = make(steps=K)
    fuse = int(os.environ.get("MPM_FUSE", "0"))
    sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=K, fuse_g2p2g=fuse))
    sim.set_scene(sc)
    m = sc.mass.reshape(-1).astype(np.float64)
    seed = np.zeros((sc.n, sc.dim), np.float32)
    seed[:, 0] = m / m.sum()
    for _ in range(2):
        sim.rewind(0)
        sim.forward(K)
        sim.backward(seed)
    sim.set_profiling(True)
    sim.rewind(0)
    sim.forward(K)
    sim.backward(seed)
    prof = sim.profile()
    tot = sum(v[0] for v in prof.values())
    out = {k: round(1e3 * v[0] / max(v[1], 1), 2) for k, v in prof.items() if v[1]}
    print(json.dumps({"lib": os.path.basename(mpm.LIB_PATH), "fuse": fuse, "us_per_launch": out,
                      "us_per_FB_step": round(1e3 * tot / K, 1)}))


if __name__ == "__main__":
    main()
