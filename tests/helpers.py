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
