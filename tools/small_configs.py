"""Rates of the small BASELINE configs ("Small configs (C1-C3 single rollout) fit in
L2, and launch latency dominates.  Report their rates"): forward and forward+backward
particle-steps/s over each config's own horizon, CUDA events on the library's stream.
  python tools/small_configs.py > profiles/r01_small_configs.jsonl"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1810_01054_b200 import mpm, scenes  # noqa: E402

CASES = [("C1 configs[0] 2D block", scenes.block_2d, 50), ("C2 configs[1] 2D walker", scenes.walker_2d, 500),
         ("C3 configs[2] 3D quadruped", scenes.quadruped_3d, 200)]


FUSE = int(os.environ.get("MPM_FUSE", "1"))  # fused G2P2G forward (NEXT N2), bench.py's default
GRAPHS = int(os.environ.get("MPM_GRAPHS", "0"))  # replay the step loops as CUDA graphs (mpm_set_graphs)


def main():
    stream = torch.cuda.Stream() if GRAPHS else torch.cuda.current_stream()  # graphs: a capturable stream
    for name, make, T in CASES:
        sc = make(steps=T)
        sim = mpm.MPM(mpm.Config.from_scene(sc, max_steps=T, stream=stream.cuda_stream, fuse_g2p2g=FUSE))
        sim.set_scene(sc)
        if GRAPHS:
            sim.set_graphs(True)
        m = sc.mass.reshape(-1).astype(np.float64)
        seed = np.zeros((sc.n, sc.dim), np.float32)
        seed[:, 0] = (m / m.sum()).astype(np.float32)
        for _ in range(2):
            sim.rewind(0)
            sim.forward(T)
            sim.backward(seed)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        sim.rewind(0)
        torch.cuda.synchronize()
        e[0].record(stream)
        sim.forward(T)
        e[1].record(stream)
        sim.backward(seed)
        e[2].record(stream)
        torch.cuda.synchronize()
        f, fb = e[0].elapsed_time(e[1]), e[0].elapsed_time(e[2])
        print(json.dumps({"config": name, "fuse_g2p2g": FUSE, "graphs": GRAPHS, "particles": sc.n, "steps": T,
                          "fwd_us_per_step": round(1e3 * f / T, 2), "fb_us_per_step": round(1e3 * fb / T, 2),
                          "fwd_particle_steps_per_s": sc.n * T / (f * 1e-3),
                          "fb_particle_steps_per_s": sc.n * T / (fb * 1e-3)}), flush=True)
        sim.close()


if __name__ == "__main__":
    main()
