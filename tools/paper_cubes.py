"""The paper's own speed workload (Table I, "a simple falling cube" P:214):
cubes of 20^3, 40^3 and 80^3 particles (8 per cell), forward and backward time per step on
this GPU, next to the paper's GTX 1080 Ti numbers (context, not a target: BASELINE.md).
Grid resolution, dt, E, nu are not printed in the paper; the cube falls from rest at res 64
(20^3, 40^3) / 128 (80^3) with the C4 recipe otherwise.  One JSON line per cube.
  python tools/paper_cubes.py [steps]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1810_01054_b200 import mpm, scenes  # noqa: E402

PAPER_MS = {20: (0.392, 0.406), 40: (1.594, 1.774), 80: (10.501, 11.594)}  # Table I (F, B) per frame


FUSE = int(os.environ.get("MPM_FUSE", "1"))  # fused G2P2G forward (NEXT N2), bench.py's default


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    stream = torch.cuda.current_stream()
    for n in (20, 40, 80):
        c = n // 2
        res = 64 if n < 80 else 128
        sc = scenes.slab_3d(steps=K, cells=(c, c, c), res=res, y0=res // 4)
        sc.v[..., 1] = 0.0  # falls from rest under gravity
        sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=K, stream=stream.cuda_stream, fuse_g2p2g=FUSE))
        sim.set_scene(sc)
        seed = np.zeros((sc.n, 3), np.float32)
        seed[:, 0] = 1.0 / sc.n
        for _ in range(2):  # warm-up
            sim.rewind(0)
            sim.forward(K)
            sim.backward(seed)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        sim.rewind(0)
        torch.cuda.synchronize()
        e[0].record(stream)
        sim.forward(K)
        e[1].record(stream)
        sim.backward(seed)
        e[2].record(stream)
        torch.cuda.synchronize()
        f = e[0].elapsed_time(e[1]) / K
        b = e[1].elapsed_time(e[2]) / K
        pf, pb = PAPER_MS[n]
        print(json.dumps({"cube": f"{n}^3 particles", "fuse_g2p2g": FUSE, "particles": sc.n, "res": res, "steps": K,
                          "fwd_ms_per_step": round(f, 4), "bwd_ms_per_step": round(b, 4),
                          "fwd_particle_steps_per_s": sc.n / (f * 1e-3), "bwd_particle_steps_per_s": sc.n / (b * 1e-3),
                          "paper_1080ti_ms_per_frame": {"fwd": pf, "bwd": pb},
                          "speedup_vs_paper_1_step_per_frame": {"fwd": round(pf / f, 1), "bwd": round(pb / b, 1)}}),
              flush=True)
        sim.close()


if __name__ == "__main__":
    main()
