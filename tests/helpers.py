"""Test-side glue: scene (fp32 arrays) -> oracle inputs (fp64 of the same fp32 values)."""
from __future__ import annotations

import numpy as np

import oracle


def oracle_cfg(scene, **over) -> oracle.Config:
    kw = dict(dim=scene.dim, res=scene.res, dt=scene.dt, gravity=tuple(scene.gravity),
              bound=scene.bound, friction=tuple(scene.friction), act_strength=scene.act_strength,
              n_act=scene.n_act)
    kw.update(over)
    return oracle.Config(**kw)


def oracle_state(scene, r: int = 0) -> np.ndarray:
    return oracle.pack(scene.x[r], scene.v[r], scene.C[r], scene.F[r])


def oracle_params(scene, r: int = 0):
    return (scene.mass[r].astype(np.float64), scene.vol[r].astype(np.float64),
            scene.E[r].astype(np.float64), scene.nu[r].astype(np.float64),
            scene.actuator_id[r], scene.act[r].astype(np.float64))


def run_oracle(scene, r: int = 0, steps=None, **over):
    cfg = oracle_cfg(scene, **over)
    m, vol, E, nu, aid, act = oracle_params(scene, r)
    T = scene.steps if steps is None else steps
    traj = oracle.forward(cfg, oracle_state(scene, r), m, vol, E, nu, aid, act[:max(T, 1)], T)
    return cfg, traj


def rel_err(a, b) -> float:
    """Norm-wise relative error ||a - b|| / ||b|| (reading R16)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def ang_mom(x, v, Cm, mass, dx):
    """Augmented APIC angular momentum sum_p m_p [x_p x v_p + (dx^2/4) eps:C_p^T]."""
    d = x.shape[1]
    if d == 2:
        return float(np.sum(mass * (x[:, 0] * v[:, 1] - x[:, 1] * v[:, 0]
                                    + dx * dx / 4 * (Cm[:, 1, 0] - Cm[:, 0, 1]))))
    L = np.cross(x, v)
    spin = np.stack([Cm[:, 2, 1] - Cm[:, 1, 2], Cm[:, 0, 2] - Cm[:, 2, 0],
                     Cm[:, 1, 0] - Cm[:, 0, 1]], axis=1)
    return (mass[:, None] * (L + dx * dx / 4 * spin)).sum(0)


# Element-wise bar for gradients, next to the norm-wise one of R16: the largest per-element
# deviation measured against the field's own scale (max |b| over the field), so that a wrong
# adjoint on a handful of particles (a wall corner, a fused-step escapee, a slab window) cannot
# hide inside a norm over 10^4-10^6 particles.  DESIGN.md section 9 records the measured margins.
ELEM_TOL = 1e-3


def elem_err(a, b) -> float:
    """max_i |a_i - b_i| / max_i |b_i| (element-wise, field scale)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    sb = np.abs(b).max() if b.size else 0.0
    if sb == 0.0:
        return float(np.abs(a).max()) if a.size else 0.0
    return float(np.abs(a - b).max() / sb)


def grad_errs(pairs):
    """{name: (norm-wise, element-wise)} for (name, gpu, oracle) triples."""
    return {k: (rel_err(a, b), elem_err(a, b)) for k, a, b in pairs}


def assert_grads(pairs, tol=1e-3, etol=ELEM_TOL, ctx=None):
    """Both bars on every gradient field: norm-wise < tol (R16) and element-wise < etol."""
    errs = grad_errs(pairs)
    bad = {k: e for k, e in errs.items() if not (e[0] < tol and e[1] < etol)}
    assert not bad, (bad, ctx)
    return errs


def wall_scenes(d, T):
    """Blocks driven into the wall bands of every kind, friction per wall (-x, +x, -y, +y, -z,
    +z) = (sticky, 2, 1, 0.5, 2, sticky): R6's c < 0 and step L's full stop (R = l_t + c l_n < 0,
    P:618/P:621, with H(R) = 0 in the adjoint) next to the sliding case."""
    from paper_1810_01054_b200 import scenes
    fr = (-1.0, 2.0, 1.0, 0.5, 2.0, -1.0)[:2 * d] + (0.0,) * (6 - 2 * d)
    lo = scenes.tiny(d, seed=77 + d, res=32, n_cells=(9,) * d, center=(2,) * d, steps=T, K=2, s=30.0,
                     friction=fr, v0=(-1.5,) * d, gravity=(-5.0,) * d)
    hi = scenes.tiny(d, seed=79 + d, res=32, n_cells=(9,) * d, center=(20,) * d, steps=T, K=2, s=30.0,
                     friction=fr, v0=(1.5,) * d, gravity=(5.0,) * d)
    return [(f"{d}D block driven into the low walls (sticky -x, c=1 -y, c=2 -z), {T} steps", lo),
            (f"{d}D block driven into the high walls (c=2 +x, c=0.5 +y, sticky +z), {T} steps", hi)]
