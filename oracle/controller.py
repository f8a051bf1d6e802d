"""Oracle of NEXT N1: the closed-loop controller embedded in P2G (Fig. 2 caption P:84,
P:279; SPEC.md observe / act / controller_adjoint).

TEST INFRASTRUCTURE ONLY (same rules as the package: only tests/, smoke() and bench.py's CPU
legs may use it).  Plain numpy for the controller, the fp64 C oracle for the MLS-MPM steps;
no blocking or reordering beyond the paper's statement.

  z_t = [target, CoM_0 .. CoM_{K-1}, V_0 .. V_{K-1}]      ("target position, the center of
        CoM_k = sum_{p in k} m_p x_p / M_k,                mass position, and velocity of each
        V_k   = sum_{p in k} m_p v_p / M_k                 composed soft component"; reading R20:
                                                            component k = actuator group k)
  a_t = tanh(W z_t + b), reshaped [K][d] -> sigma_pa (R4)

Reverse (SPEC controller_adjoint, derived by the chain rule): with g_a = dL/da_t from step K
 of the same time step,
  g_pre = g_a * (1 - a_t^2);  dL/dW += g_pre z_t^T;  dL/db += g_pre;  dL/dz = W^T g_pre,
and dL/dz flows into dL/dx_p, dL/dv_p of state t through the group means (m_p / M_k).
"""
from __future__ import annotations

import numpy as np

import oracle


def n_obs(d: int, K: int) -> int:
    """Length of z: target (d) + K CoMs (d each) + K mean velocities (d each)."""
    return d * (1 + 2 * K)


def observe(x, v, mass, act_id, K, target):
    """z = concat(target, per-group mass-weighted CoM, per-group mass-weighted mean velocity)."""
    x = np.asarray(x, np.float64)
    v = np.asarray(v, np.float64)
    m = np.asarray(mass, np.float64)
    com, vel = [], []
    for k in range(K):
        sel = np.asarray(act_id) == k
        if not sel.any():
            raise ValueError(f"empty actuator group {k}")
        M = m[sel].sum()
        com.append((m[sel, None] * x[sel]).sum(0) / M)
        vel.append((m[sel, None] * v[sel]).sum(0) / M)
    return np.concatenate([np.asarray(target, np.float64)] + com + vel)


def act(W, b, z):
    """a = tanh(W z + b)."""
    return np.tanh(np.asarray(W, np.float64) @ z + np.asarray(b, np.float64))


def forward(cfg, state0, mass, vol, E, nu, act_id, W, b, target, n_steps):
    """Closed-loop rollout: returns (traj [(T+1)][n][S], actuation [T][K][d], z [T][nz])."""
    d, K = cfg.dim, cfg.n_act
    traj = [np.asarray(state0, np.float64)]
    acts, zs = [], []
    for t in range(n_steps):
        x, v, _, _ = oracle.unpack(traj[t], d)
        z = observe(x, v, mass, act_id, K, target)
        a = act(W, b, z).reshape(K, d)
        traj.append(oracle.forward(cfg, traj[t], mass, vol, E, nu, act_id, a[None], 1)[1])
        acts.append(a)
        zs.append(z)
    return np.stack(traj), np.stack(acts), np.stack(zs)


def backward(cfg, traj, mass, vol, E, nu, act_id, W, b, acts, zs, seed):
    """Reverse mode of the closed-loop rollout from dL/dstate_T = seed.
    Returns (dL/dstate_0, dL/dE, dL/dnu, dL/dW, dL/db, dL/dtarget, dL/da [T][K][d])."""
    d, K = cfg.dim, cfg.n_act
    T = traj.shape[0] - 1
    W = np.asarray(W, np.float64)
    m = np.asarray(mass, np.float64)
    aid = np.asarray(act_id)
    g = np.asarray(seed, np.float64).copy()
    gE = np.zeros(len(m))
    gnu = np.zeros(len(m))
    gW = np.zeros_like(W)
    gb = np.zeros(W.shape[0])
    gtarget = np.zeros(d)
    ga_all = np.zeros((T, K, d))
    for t in reversed(range(T)):
        # the MLS-MPM step t (steps A-L) with the actuation the controller produced
        g0, gE_t, gnu_t, ga_t = oracle.backward(cfg, traj[t:t + 2], mass, vol, E, nu, act_id,
                                                acts[t][None], g)
        ga_all[t] = ga_t[0]
        # controller adjoint
        a = acts[t].reshape(-1)
        gpre = ga_t[0].reshape(-1) * (1.0 - a * a)
        gW += np.outer(gpre, zs[t])
        gb += gpre
        gz = W.T @ gpre
        # observe adjoint: z = [target, CoM_k, V_k]
        gtarget += gz[:d]
        for k in range(K):
            sel = aid == k
            M = m[sel].sum()
            g0[sel, 0:d] += (m[sel] / M)[:, None] * gz[d + k * d:d + (k + 1) * d]
            g0[sel, d:2 * d] += (m[sel] / M)[:, None] * gz[d + K * d + k * d:d + K * d + (k + 1) * d]
        g = g0
        gE += gE_t
        gnu += gnu_t
    return g, gE, gnu, gW, gb, gtarget, ga_all
