"""Seeded synthetic scenes shaped like the paper's workloads.

This module is the ONLY code shared by the CUDA path's callers and the oracle's callers.
It holds no arithmetic of the method (no kernel, stress, transfer or adjoint): it only
samples particles on jittered lattices and fills parameter arrays.  numpy only.

Common recipe: domain [0,1)^d, dx = 1/res, 2^d particles per cell on a
jittered sub-cell lattice (uniform jitter inside each sub-cell), V0 = dx^d / 2^d,
m = rho * V0 with rho = 1, E = 1e3, nu = 0.3, gravity -9.8 e_y, wall band 3 nodes,
floor friction c = 0.5, other walls c = 0.  dt is below the CFL bound of P:380
(dt <= C dx sqrt(rho/E), C = 0.5).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Scene:
    name: str
    dim: int
    res: int
    dt: float
    steps: int
    gravity: tuple
    bound: int
    friction: tuple
    act_strength: float
    n_act: int
    # per rollout arrays, leading dim = batch
    x: np.ndarray          # [B][N][d] float32
    v: np.ndarray          # [B][N][d] float32
    F: np.ndarray          # [B][N][d][d] float32
    C: np.ndarray          # [B][N][d][d] float32
    mass: np.ndarray       # [B][N] float32
    vol: np.ndarray        # [B][N] float32
    E: np.ndarray          # [B][N] float32
    nu: np.ndarray         # [B][N] float32
    actuator_id: np.ndarray  # [B][N] int32 (-1 = none)
    act: np.ndarray        # [B][T][K][d] float32
    meta: dict = field(default_factory=dict)

    @property
    def batch(self) -> int:
        return self.x.shape[0]

    @property
    def n(self) -> int:
        return self.x.shape[1]


def _lattice(dim, res, boxes, rng, jitter=1.0):
    """boxes: list of (lo_cell[d], hi_cell[d], tag).  Returns positions [N][d] and tags."""
    dx = 1.0 / res
    pos, tags = [], []
    sub = np.array(np.meshgrid(*([np.arange(2)] * dim), indexing="ij")).reshape(dim, -1).T
    for lo, hi, tag in boxes:
        axes = [np.arange(lo[a], hi[a]) for a in range(dim)]
        cells = np.array(np.meshgrid(*axes, indexing="ij")).reshape(dim, -1).T
        p = (cells[:, None, :] + (sub[None, :, :] + 0.5 + jitter * (rng.random((len(cells), len(sub), dim)) - 0.5)) * 0.5) * dx
        pos.append(p.reshape(-1, dim))
        tags.append(np.full(len(cells) * len(sub), tag, np.int32))
    return np.concatenate(pos).astype(np.float32), np.concatenate(tags)


def _common(dim, res, x, rng, E=1e3, nu=0.3, rho=1.0):
    n = x.shape[0]
    dx = 1.0 / res
    vol = np.full(n, dx ** dim / 2 ** dim, np.float32)
    mass = (rho * vol).astype(np.float32)
    return (mass, vol, np.full(n, E, np.float32), np.full(n, nu, np.float32))


def _pack(name, dim, res, dt, steps, K, s, xs, vs, Fs, Cs, ms, vols, Es, nus, aids, acts,
          gravity=None, friction=None, bound=3, meta=None):
    g = gravity if gravity is not None else ((0.0, -9.8) if dim == 2 else (0.0, -9.8, 0.0))
    f = friction if friction is not None else (0.0, 0.0, 0.5, 0.0, 0.0, 0.0)
    return Scene(name, dim, res, dt, steps, tuple(g), bound, tuple(f), s, K,
                 np.stack(xs), np.stack(vs), np.stack(Fs), np.stack(Cs), np.stack(ms),
                 np.stack(vols), np.stack(Es), np.stack(nus), np.stack(aids), np.stack(acts),
                 meta or {})


def _identity(n, d):
    return np.broadcast_to(np.eye(d, dtype=np.float32), (n, d, d)).copy()


def block_2d(seed=0, batch=1, steps=50, perturb=False):
    """C1 (configs[0]): 2D 64^2 grid, 16x16-cell elastic block, 1,024 particles, v0 = (1, 0.5)
    + 0.1 N(0,1); never reaches the wall bands in 50 steps (closed-form CoM gradient holds)."""
    dim, res = 2, 64
    xs, vs, Fs, Cs, ms, vols, Es, nus, aids, acts = ([] for _ in range(10))
    for r in range(batch):
        rng = np.random.default_rng(seed + r)
        x, _ = _lattice(dim, res, [((24, 24), (40, 40), 0)], rng)
        n = x.shape[0]
        v = (np.array([1.0, 0.5]) + 0.1 * rng.standard_normal((n, dim))).astype(np.float32)
        F = _identity(n, dim)
        Cm = np.zeros((n, dim, dim), np.float32)
        if perturb:
            F = (F + 0.05 * rng.standard_normal((n, dim, dim))).astype(np.float32)
            Cm = (5.0 * rng.standard_normal((n, dim, dim))).astype(np.float32)
        m, vol, E, nu = _common(dim, res, x, rng)
        xs.append(x); vs.append(v); Fs.append(F); Cs.append(Cm); ms.append(m); vols.append(vol)
        Es.append(E); nus.append(nu); aids.append(np.full(n, -1, np.int32))
        acts.append(np.zeros((steps, 1, dim), np.float32))
    return _pack("C1_block2d", dim, res, 2e-4, steps, 0, 0.0, xs, vs, Fs, Cs, ms, vols, Es, nus,
                 aids, acts)


def walker_2d(seed=0, batch=1, steps=500):
    """C2 (configs[1]): 2D 128^2 walker, body 40x14 cells on 4 legs of 8x28 cells standing on
    the floor; 5,824 particles; K = 4 leg actuators on the vertical channel,
    a[t][k] = sin(2 pi t / 100 + k pi / 2), s = 40 (s = 300 inverts elements within 500 steps)."""
    dim, res, K = 2, 128, 4
    legs_x = (20, 31, 41, 52)
    xs, vs, Fs, Cs, ms, vols, Es, nus, aids, acts = ([] for _ in range(10))
    for r in range(batch):
        rng = np.random.default_rng(seed + r)
        boxes = [((20, 31), (60, 45), -1)] + [((lx, 3), (lx + 8, 31), k) for k, lx in enumerate(legs_x)]
        x, tag = _lattice(dim, res, boxes, rng)
        n = x.shape[0]
        m, vol, E, nu = _common(dim, res, x, rng)
        t = np.arange(steps)[:, None]
        k = np.arange(K)[None, :]
        a = np.zeros((steps, K, dim), np.float32)
        a[:, :, 1] = np.sin(2 * np.pi * t / 100 + k * np.pi / 2 + r * 0.1)
        xs.append(x); vs.append(np.zeros((n, dim), np.float32)); Fs.append(_identity(n, dim))
        Cs.append(np.zeros((n, dim, dim), np.float32)); ms.append(m); vols.append(vol)
        Es.append(E); nus.append(nu); aids.append(tag.astype(np.int32)); acts.append(a)
    return _pack("C2_walker2d", dim, res, 1e-4, steps, K, 40.0, xs, vs, Fs, Cs, ms, vols, Es,
                 nus, aids, acts)


def quadruped_3d(seed=0, batch=1, steps=200, e_scale=False):
    """C3 (configs[2]): 3D 64^3 quadruped, body 24x6x12 cells + 4 legs 6x14x6 cells;
    29,952 particles; K = 16 (each leg split 2x2 in x-z, "up to 16 actuators").
    C5b uses batch=64 with per-rollout phases and an E scale U(0.5, 2) (e_scale=True)."""
    dim, res, K = 3, 64, 16
    legs = [(20, 20), (38, 20), (20, 26), (38, 26)]  # (x, z) lower corners of 6x6 legs
    xs, vs, Fs, Cs, ms, vols, Es, nus, aids, acts = ([] for _ in range(10))
    for r in range(batch):
        rng = np.random.default_rng(seed + r)
        boxes = [((20, 17, 20), (44, 23, 32), -1)]
        for li, (lx, lz) in enumerate(legs):
            for qx in range(2):
                for qz in range(2):
                    lo = (lx + 3 * qx, 3, lz + 3 * qz)
                    boxes.append((lo, (lo[0] + 3, 17, lo[2] + 3), li * 4 + qx * 2 + qz))
        x, tag = _lattice(dim, res, boxes, rng)
        n = x.shape[0]
        scale = rng.uniform(0.5, 2.0) if e_scale else 1.0
        m, vol, E, nu = _common(dim, res, x, rng, E=1e3 * scale)
        t = np.arange(steps)[:, None]
        k = np.arange(K)[None, :]
        ph = rng.uniform(0, 2 * np.pi) if batch > 1 else 0.0
        a = np.zeros((steps, K, dim), np.float32)
        a[:, :, 1] = np.sin(2 * np.pi * t / 100 + k * np.pi / 8 + ph)
        xs.append(x); vs.append(np.zeros((n, dim), np.float32)); Fs.append(_identity(n, dim))
        Cs.append(np.zeros((n, dim, dim), np.float32)); ms.append(m); vols.append(vol)
        Es.append(E); nus.append(nu); aids.append(tag.astype(np.int32)); acts.append(a)
    return _pack("C3_quadruped3d", dim, res, 2e-4, steps, K, 100.0, xs, vs, Fs, Cs, ms, vols,
                 Es, nus, aids, acts)


def slab_3d(seed=0, batch=1, steps=100, cells=(64, 32, 64), res=128, y0=5, dt=1e-4, name="C4_slab3d"):
    """C4 (configs[3]): 3D 128^3 falling neo-Hookean slab of 64x32x64 cells (x, y, z),
    1,048,576 particles, v0 = (0, -1, 0); K = 8 octant actuators, sinusoidal."""
    dim, K = 3, 8
    lo = ((res - cells[0]) // 2, y0, (res - cells[2]) // 2)
    hi = (lo[0] + cells[0], lo[1] + cells[1], lo[2] + cells[2])
    xs, vs, Fs, Cs, ms, vols, Es, nus, aids, acts = ([] for _ in range(10))
    for r in range(batch):
        rng = np.random.default_rng(seed + r)
        x, _ = _lattice(dim, res, [(lo, hi, 0)], rng)
        n = x.shape[0]
        mid = ((np.array(lo) + np.array(hi)) * 0.5 / res).astype(np.float32)
        oct_id = ((x[:, 0] >= mid[0]).astype(np.int32) * 4 + (x[:, 1] >= mid[1]) * 2
                  + (x[:, 2] >= mid[2])).astype(np.int32)
        m, vol, E, nu = _common(dim, res, x, rng)
        t = np.arange(steps)[:, None]
        k = np.arange(K)[None, :]
        a = np.zeros((steps, K, dim), np.float32)
        a[:, :, 1] = np.sin(2 * np.pi * t / 50 + k * np.pi / 4)
        v = np.zeros((n, dim), np.float32)
        v[:, 1] = -1.0
        xs.append(x); vs.append(v); Fs.append(_identity(n, dim))
        Cs.append(np.zeros((n, dim, dim), np.float32)); ms.append(m); vols.append(vol)
        Es.append(E); nus.append(nu); aids.append(oct_id); acts.append(a)
    return _pack(name, dim, res, dt, steps, K, 100.0, xs, vs, Fs, Cs, ms, vols, Es,
                 nus, aids, acts)


def slab_c5a(seed=0, steps=100):
    """C5a (configs[4]): 3D 256^3 slab of 240x32x136 cells, 8,355,840 particles,
    dt = 5e-5, the C4 recipe otherwise; sharded by x-slab across GPUs."""
    return slab_3d(seed=seed, steps=steps, cells=(240, 32, 136), res=256, y0=10, dt=5e-5,
                   name="C5a_slab3d")


def tiny(dim, seed=0, n_cells=None, res=None, steps=10, perturb=True, gravity=None,
         friction=None, K=2, s=50.0, center=None, v0=None, E=1e3, jitter=1.0):
    """Small fp64-checkable scenes for parity and finite differences: a block of cells
    (default 3x3 in 2D at res 16, 3x3x3 in 3D at res 8... 16) with random F0, C0 (SURVEY 8d:
    F0 = I + 0.05 N(0,1), C0 = 5 N(0,1)) and K actuators split by particle index parity."""
    res = res or 16
    n_cells = n_cells or (3,) * dim
    rng = np.random.default_rng(seed)
    c0 = center if center is not None else tuple(res // 2 - nc // 2 for nc in n_cells)
    lo = tuple(int(c) for c in c0)
    hi = tuple(lo[a] + n_cells[a] for a in range(dim))
    x, _ = _lattice(dim, res, [(lo, hi, 0)], rng, jitter=jitter)
    n = x.shape[0]
    v = (0.3 * rng.standard_normal((n, dim))).astype(np.float32)
    if v0 is not None:
        v += np.asarray(v0, np.float32)
    F = _identity(n, dim)
    Cm = np.zeros((n, dim, dim), np.float32)
    if perturb:
        F = (F + 0.05 * rng.standard_normal((n, dim, dim))).astype(np.float32)
        Cm = (5.0 * rng.standard_normal((n, dim, dim))).astype(np.float32)
    m, vol, Ea, nu = _common(dim, res, x, rng, E=E)
    aid = (np.arange(n) % (K + 1) - 1).astype(np.int32) if K > 0 else np.full(n, -1, np.int32)
    a = (rng.standard_normal((steps, max(K, 1), dim))).astype(np.float32)
    g = gravity if gravity is not None else ((0.0, -9.8) if dim == 2 else (0.0, -9.8, 0.0))
    f = friction if friction is not None else (0.0, 0.0, 0.5, 0.0, 0.0, 0.0)
    return Scene(f"tiny{dim}d", dim, res, 1e-4, steps, tuple(g), 3, tuple(f), s, K,
                 x[None], v[None], F[None], Cm[None], m[None], vol[None], Ea[None], nu[None],
                 aid[None], a[None])


CONFIGS = {
    "C1": block_2d,
    "C2": walker_2d,
    "C3": quadruped_3d,
    "C4": slab_3d,
}
