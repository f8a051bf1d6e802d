"""The oracle's timing builds (bench.py cpu_baseline): the OpenMP build (per-chunk
scatter grids merged in fixed chunk order) and the fp32 build against the serial fp64 oracle.
They add no arithmetic of the method -- the same per-particle / per-node functions in
parallel loops -- so the OpenMP fp64 result equals the serial one up to the summation order
of the node sums, and the fp32 one to fp32 rounding."""
import os

os.environ.setdefault("OMP_NUM_THREADS", "4")

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1810_01054_b200 import scenes  # noqa: E402
from tests.helpers import oracle_cfg, oracle_params, oracle_state, rel_err  # noqa: E402


def _scene(d):
    return scenes.tiny(d, seed=40 + d, res=32 if d == 2 else 16, n_cells=(10, 7) if d == 2 else (6, 5, 4),
                       steps=5, K=2, s=40.0, friction=(0.5, -1.0, 2.0, 0.3, 1.0, 0.0))


def test_omp_and_fp32_builds_match_the_serial_oracle():
    for d in (2, 3):
        sc = _scene(d)
        T = sc.steps
        cfg = oracle_cfg(sc)
        m, vol, E, nu, aid, act = oracle_params(sc)
        st = oracle_state(sc)
        traj = oracle.forward(cfg, st, m, vol, E, nu, aid, act[:T], T)
        seed = np.random.default_rng(d).standard_normal(traj[T].shape)
        g0, *_ = oracle.backward(cfg, traj, m, vol, E, nu, aid, act[:T], seed)
        _, _, s64 = oracle.forward_backward_timing(cfg, st, m, vol, E, nu, aid, act[:T], seed, T, "serial64")
        np.testing.assert_array_equal(s64, g0)  # same source, same order
        _, _, o64 = oracle.forward_backward_timing(cfg, st, m, vol, E, nu, aid, act[:T], seed, T, "omp64")
        assert rel_err(o64, g0) < 1e-12
        for v in ("serial32", "omp32"):
            _, _, g32 = oracle.forward_backward_timing(cfg, st, m, vol, E, nu, aid, act[:T], seed, T, v)
            assert rel_err(g32, g0) < 1e-3, (v, rel_err(g32, g0))
    assert oracle.omp_threads() >= 1
