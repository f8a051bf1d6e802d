"""CPU oracle for the differentiable MLS-MPM step (ChainQueen, arXiv 1810.01054).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_1810_01054_b200``) never imports it and shares no code with it.

The arithmetic lives in ``mpm_oracle.c`` (plain C99, fp64); this module only builds that
file with gcc and marshals numpy arrays through ctypes.  See ``mpm_oracle.h`` for the
citations of every function (PAPER.md lines and DESIGN.md readings).

State record per particle (S = 2d + 2d^2 doubles): x[d], v[d], C[d][d], F[d][d].
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# tools/mutation_check.py points this at a mutated build of mpm_oracle.c (never the product)
_LIB_OVERRIDE = os.environ.get("MPM_ORACLE_LIB")

ORC_OK, ORC_ERR_OUT_OF_DOMAIN, ORC_ERR_INVERTED, ORC_ERR_ARG = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile mpm_oracle.c into liboracle.so (gcc, -O2, no fast-math, no FP contraction)."""
    if _LIB_OVERRIDE:
        return _LIB_OVERRIDE
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "mpm_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
             "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cfg(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("res", C.c_int), ("n", C.c_int), ("n_act", C.c_int),
        ("dt", C.c_double), ("gravity", C.c_double * 3), ("bound", C.c_int),
        ("friction", C.c_double * 6), ("act_strength", C.c_double), ("eps", C.c_double),
        ("material", C.c_int),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        fp = C.POINTER(C.c_float)
        L.orc_N.restype = C.c_double
        L.orc_N.argtypes = [C.c_double]
        L.orc_dN.restype = C.c_double
        L.orc_dN.argtypes = [C.c_double]
        L.orc_weights.argtypes = [C.c_double, ip, dp, dp]
        L.orc_det.restype = C.c_double
        L.orc_det.argtypes = [C.c_int, dp]
        L.orc_psi.restype = C.c_double
        L.orc_psi.argtypes = [C.c_int, dp, C.c_double, C.c_double]
        L.orc_pk1.argtypes = [C.c_int, dp, C.c_double, C.c_double, dp]
        L.orc_dPdF.argtypes = [C.c_int, dp, C.c_double, C.c_double, dp]
        L.orc_psi_fcr.restype = C.c_double
        L.orc_psi_fcr.argtypes = [C.c_int, dp, C.c_double, C.c_double]
        L.orc_pk1_fcr.argtypes = [C.c_int, dp, C.c_double, C.c_double, dp]
        L.orc_dPdF_fcr.argtypes = [C.c_int, dp, C.c_double, C.c_double, dp]
        L.orc_polar.argtypes = [C.c_int, dp, dp]
        L.orc_lame.argtypes = [C.c_double, C.c_double, dp, dp]
        L.orc_project.argtypes = [C.c_int, dp, dp, C.c_double, C.c_double, dp]
        L.orc_project_adj.argtypes = [C.c_int, dp, dp, C.c_double, C.c_double, dp, dp]
        L.orc_grid_node.argtypes = [C.POINTER(_Cfg), ip, C.c_double, dp, dp, dp]
        L.orc_grid_node_adj.argtypes = [C.POINTER(_Cfg), ip, C.c_double, dp, dp, dp, dp]
        L.orc_step_grid.restype = C.c_int
        L.orc_step_grid.argtypes = [C.POINTER(_Cfg), dp, dp, dp, dp, dp, ip, dp, dp, dp, dp, dp]
        L.orc_forward.restype = C.c_int
        L.orc_forward.argtypes = [C.POINTER(_Cfg), C.c_int, dp, dp, dp, dp, dp, ip, dp, ip]
        L.orc_backward.restype = C.c_int
        L.orc_backward.argtypes = [C.POINTER(_Cfg), C.c_int, dp, dp, dp, dp, dp, ip, dp, dp,
                                   dp, dp, dp, dp]
        L.orc_backward_ex.restype = C.c_int
        L.orc_backward_ex.argtypes = [C.POINTER(_Cfg), C.c_int, dp, dp, dp, dp, dp, ip, dp, dp,
                                      dp, dp, dp, dp, dp]
        L.orc_bin.restype = C.c_int
        L.orc_bin.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, fp, ip, ip, ip]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _f(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _dv(x, n=None):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return a


@dataclass
class Config:
    """Oracle configuration of one rollout (mirrors the fields the paper's step needs)."""
    dim: int
    res: int
    dt: float
    gravity: tuple = (0.0, 0.0, 0.0)
    bound: int = 3
    friction: tuple = (0.0, 0.0, 0.0, 0.0, 0.0, 0.0)
    act_strength: float = 0.0
    n_act: int = 0
    eps: float = 1e-10  # R7
    material: int = 0   # 0 = neo-Hookean (R1), 1 = fixed-corotated (R21)

    def c(self, n: int) -> _Cfg:
        g = list(self.gravity) + [0.0] * (3 - len(self.gravity))
        f = list(self.friction) + [0.0] * (6 - len(self.friction))
        return _Cfg(self.dim, self.res, n, self.n_act, self.dt, (C.c_double * 3)(*g[:3]),
                    self.bound, (C.c_double * 6)(*f[:6]), self.act_strength, self.eps, self.material)


class OracleError(RuntimeError):
    def __init__(self, code, where=None):
        self.code = code
        self.where = where
        super().__init__(f"oracle error {code} at {where}")


def S_of(d: int) -> int:
    return 2 * d + 2 * d * d


def pack(x, v, Cm, F) -> np.ndarray:
    """[n][d], [n][d], [n][d][d], [n][d][d] -> [n][S] records."""
    x = np.asarray(x, np.float64)
    n, d = x.shape
    return np.ascontiguousarray(np.concatenate(
        [x, np.asarray(v, np.float64).reshape(n, d), np.asarray(Cm, np.float64).reshape(n, d * d),
         np.asarray(F, np.float64).reshape(n, d * d)], axis=1))


def unpack(rec: np.ndarray, d: int):
    n = rec.shape[-2]
    lead = rec.shape[:-2]
    x = rec[..., 0:d]
    v = rec[..., d:2 * d]
    Cm = rec[..., 2 * d:2 * d + d * d].reshape(*lead, n, d, d)
    F = rec[..., 2 * d + d * d:].reshape(*lead, n, d, d)
    return x, v, Cm, F


def forward(cfg: Config, state0: np.ndarray, mass, vol, E, nu, act_id=None, act=None,
            n_steps: int = 1) -> np.ndarray:
    """Run n_steps; returns the trajectory [(n_steps+1)][n][S] (P:165 memo)."""
    state0 = np.asarray(state0, np.float64)
    n, S = state0.shape
    assert S == S_of(cfg.dim)
    traj = np.zeros((n_steps + 1, n, S))
    traj[0] = state0
    mass, vol, E, nu = (_dv(a) for a in (mass, vol, E, nu))
    aid = np.ascontiguousarray(np.full(n, -1, np.int32) if act_id is None else np.asarray(act_id, np.int32))
    if act is None:
        act = np.zeros((max(n_steps, 1), max(cfg.n_act, 1), cfg.dim))
    act = _dv(act)
    err_idx = np.zeros(2, np.int32)
    cc = cfg.c(n)
    rc = lib().orc_forward(C.byref(cc), n_steps, _d(traj), _d(mass), _d(vol), _d(E), _d(nu),
                           _i(aid), _d(act), _i(err_idx))
    if rc:
        raise OracleError(rc, tuple(err_idx))
    return traj


def step_grid(cfg: Config, state: np.ndarray, mass, vol, E, nu, act_id=None, act_t=None):
    """Grid of one step: (m [res^d], p, vbar, v [res^d][d]) -- P2G then grid operation."""
    state = np.ascontiguousarray(state, np.float64)
    n = state.shape[0]
    d = cfg.dim
    nn = cfg.res ** d
    mass, vol, E, nu = (_dv(a) for a in (mass, vol, E, nu))
    aid = np.ascontiguousarray(np.full(n, -1, np.int32) if act_id is None else np.asarray(act_id, np.int32))
    act_t = _dv(np.zeros((max(cfg.n_act, 1), d)) if act_t is None else act_t)
    m = np.zeros(nn); p = np.zeros((nn, d)); vbar = np.zeros((nn, d)); v = np.zeros((nn, d))
    cc = cfg.c(n)
    rc = lib().orc_step_grid(C.byref(cc), _d(state), _d(mass), _d(vol), _d(E), _d(nu), _i(aid),
                             _d(act_t), _d(m), _d(p), _d(vbar), _d(v))
    if rc:
        raise OracleError(rc)
    return m, p, vbar, v


def backward(cfg: Config, traj: np.ndarray, mass, vol, E, nu, act_id=None, act=None,
             seed=None):
    """Reverse-mode from dL/dstate_T = seed.  Returns (dL/dstate_0, dL/dE, dL/dnu, dL/da)."""
    traj = np.ascontiguousarray(traj, np.float64)
    n_steps = traj.shape[0] - 1
    n, S = traj.shape[1], traj.shape[2]
    mass, vol, E, nu = (_dv(a) for a in (mass, vol, E, nu))
    aid = np.ascontiguousarray(np.full(n, -1, np.int32) if act_id is None else np.asarray(act_id, np.int32))
    K = max(cfg.n_act, 1)
    if act is None:
        act = np.zeros((max(n_steps, 1), K, cfg.dim))
    act = _dv(act)
    seed = _dv(seed)
    g0 = np.zeros((n, S))
    gE = np.zeros(n)
    gnu = np.zeros(n)
    ga = np.zeros((max(n_steps, 1), K, cfg.dim))
    cc = cfg.c(n)
    rc = lib().orc_backward(C.byref(cc), n_steps, _d(traj), _d(mass), _d(vol), _d(E), _d(nu),
                            _i(aid), _d(act), _d(seed), _d(g0), _d(gE), _d(gnu), _d(ga))
    if rc:
        raise OracleError(rc)
    return g0, gE, gnu, ga[:n_steps, :cfg.n_act]


def backward_ex(cfg: Config, traj: np.ndarray, mass, vol, E, nu, act_id=None, act=None,
                seeds=None):
    """Reverse-mode with a seed for every state (seeds [(T+1)][n][S]; a running loss) and the
    mass gradient.  Returns (dL/dstate_0, dL/dE, dL/dnu, dL/da, dL/dm)."""
    traj = np.ascontiguousarray(traj, np.float64)
    n_steps = traj.shape[0] - 1
    n, S = traj.shape[1], traj.shape[2]
    mass, vol, E, nu = (_dv(a) for a in (mass, vol, E, nu))
    aid = np.ascontiguousarray(np.full(n, -1, np.int32) if act_id is None else np.asarray(act_id, np.int32))
    K = max(cfg.n_act, 1)
    if act is None:
        act = np.zeros((max(n_steps, 1), K, cfg.dim))
    act = _dv(act)
    seeds = _dv(seeds)
    assert seeds.shape == traj.shape
    g0 = np.zeros((n, S))
    gE = np.zeros(n)
    gnu = np.zeros(n)
    gm = np.zeros(n)
    ga = np.zeros((max(n_steps, 1), K, cfg.dim))
    cc = cfg.c(n)
    rc = lib().orc_backward_ex(C.byref(cc), n_steps, _d(traj), _d(mass), _d(vol), _d(E), _d(nu),
                               _i(aid), _d(act), _d(seeds), _d(g0), _d(gE), _d(gnu), _d(ga), _d(gm))
    if rc:
        raise OracleError(rc)
    return g0, gE, gnu, ga[:n_steps, :cfg.n_act], gm


def bin_particles(dim: int, res: int, x32: np.ndarray):
    """Binning on fp32 positions x32 [B][n][d] -> (key [B*n], perm [B*n], block_start)."""
    x32 = np.ascontiguousarray(x32, np.float32)
    B, n, d = x32.shape
    Bb = 4 if dim == 3 else 8
    nb = (res // Bb) ** dim
    key = np.zeros(B * n, np.int32)
    perm = np.zeros(B * n, np.int32)
    bs = np.zeros(B * nb + 1, np.int32)
    rc = lib().orc_bin(dim, res, B, n, _f(x32), _i(key), _i(perm), _i(bs))
    if rc:
        raise OracleError(rc)
    return key, perm, bs


# ---- unit pieces -------------------------------------------------------------------
def N(u: float) -> float:
    return lib().orc_N(float(u))


def dN(u: float) -> float:
    return lib().orc_dN(float(u))


def weights(xg: float):
    base = C.c_int(0)
    w = np.zeros(3)
    dw = np.zeros(3)
    lib().orc_weights(float(xg), C.byref(base), _d(w), _d(dw))
    return base.value, w, dw


def psi(F, mu, lam, material: int = 0) -> float:
    F = _dv(F)
    f = lib().orc_psi_fcr if material == 1 else lib().orc_psi
    return f(F.shape[0], _d(F.reshape(-1).copy()), mu, lam)


def pk1(F, mu, lam, material: int = 0):
    F = _dv(F)
    d = F.shape[0]
    P = np.zeros((d, d))
    f = lib().orc_pk1_fcr if material == 1 else lib().orc_pk1
    f(d, _d(np.ascontiguousarray(F)), mu, lam, _d(P))
    return P


def dPdF(F, mu, lam, material: int = 0):
    F = _dv(F)
    d = F.shape[0]
    H = np.zeros((d, d, d, d))
    f = lib().orc_dPdF_fcr if material == 1 else lib().orc_dPdF
    f(d, _d(np.ascontiguousarray(F)), mu, lam, _d(H))
    return H


def polar(F):
    """R of the polar decomposition F = R S (fixed-corotated model, R21)."""
    F = _dv(F)
    d = F.shape[0]
    R = np.zeros((d, d))
    rc = lib().orc_polar(d, _d(np.ascontiguousarray(F)), _d(R))
    if rc:
        raise OracleError(rc)
    return R


def lame(E, nu):
    mu = C.c_double(0)
    lam = C.c_double(0)
    lib().orc_lame(E, nu, C.byref(mu), C.byref(lam))
    return mu.value, lam.value


def project(v, n, c, eps=1e-10):
    v = _dv(v)
    n = _dv(n)
    out = np.zeros_like(v)
    lib().orc_project(v.shape[0], _d(v), _d(n), c, eps, _d(out))
    return out


def project_adj(v, n, c, dvstar, eps=1e-10):
    v = _dv(v)
    n = _dv(n)
    g = _dv(dvstar)
    out = np.zeros_like(v)
    lib().orc_project_adj(v.shape[0], _d(v), _d(n), c, eps, _d(g), _d(out))
    return out


def grid_node(cfg: Config, node, m, p):
    node = np.ascontiguousarray(node, np.int32)
    p = _dv(p)
    vbar = np.zeros(cfg.dim)
    v = np.zeros(cfg.dim)
    cc = cfg.c(0)
    lib().orc_grid_node(C.byref(cc), _i(node), float(m), _d(p), _d(vbar), _d(v))
    return vbar, v


def grid_node_adj(cfg: Config, node, m, p, dv):
    node = np.ascontiguousarray(node, np.int32)
    p = _dv(p)
    dv = _dv(dv)
    dp = np.zeros(cfg.dim)
    dm = C.c_double(0)
    cc = cfg.c(0)
    lib().orc_grid_node_adj(C.byref(cc), _i(node), float(m), _d(p), _d(dv), _d(dp), C.byref(dm))
    return dp, dm.value


# ---- timing builds (bench.py cpu_baseline) -------------------------------------
# mpm_oracle_omp.c = this oracle's per-particle / per-node functions in OpenMP loops with
# per-chunk scatter grids merged in fixed chunk order; mpm_oracle_f32.c = the same compiled with
# float arithmetic.  Neither adds arithmetic of the method (tests/test_oracle_omp.py checks them
# against the serial fp64 oracle).
_OMP_LIBS = {}


def build_omp(fp32: bool = False, force: bool = False) -> str:
    src = os.path.join(_HERE, "mpm_oracle_f32.c" if fp32 else "mpm_oracle_omp.c")
    out = os.path.join(_HERE, "liboracle_omp32.so" if fp32 else "liboracle_omp.so")
    deps = [src, _SRC, os.path.join(_HERE, "mpm_oracle_omp.c"), os.path.join(_HERE, "mpm_oracle.h")]
    if force or not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(p) for p in deps):
        tmp = out + f".tmp{os.getpid()}"
        flags = ["-fsingle-precision-constant"] if fp32 else []
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
                               "-shared", *flags, "-I", _HERE, "-o", tmp, src, "-lm"])
        os.replace(tmp, out)
    return out


class _Cfg32(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("res", C.c_int), ("n", C.c_int), ("n_act", C.c_int),
        ("dt", C.c_float), ("gravity", C.c_float * 3), ("bound", C.c_int),
        ("friction", C.c_float * 6), ("act_strength", C.c_float), ("eps", C.c_float),
        ("material", C.c_int),
    ]


def _omp_lib(fp32: bool):
    if fp32 not in _OMP_LIBS:
        L = C.CDLL(build_omp(fp32))
        L.orc_omp_threads.restype = C.c_int
        _OMP_LIBS[fp32] = L
    return _OMP_LIBS[fp32]


def omp_threads() -> int:
    """Threads the OpenMP build uses (OMP_NUM_THREADS or all cores)."""
    return _omp_lib(False).orc_omp_threads()


def forward_backward_timing(cfg: Config, state0, mass, vol, E, nu, act_id, act, seed, n_steps: int,
                            variant: str = "omp64"):
    """Forward n_steps + backward from `seed` with one of the timing builds: "serial64" (the
    oracle as it stands), "serial32", "omp64", "omp32".  Returns (forward s, forward+backward s,
    dL/dstate_0).  The serial ones run the OpenMP libraries' serial entry points (orc_forward /
    orc_backward compiled there), the omp ones orc_forward_omp / orc_backward_omp."""
    import time
    fp32 = variant.endswith("32")
    L = _omp_lib(fp32)
    omp = variant.startswith("omp")
    ft = np.float32 if fp32 else np.float64
    cp = (lambda a: a.ctypes.data_as(C.POINTER(C.c_float))) if fp32 else _d
    n, S = np.asarray(state0).shape
    traj = np.zeros((n_steps + 1, n, S), ft)
    traj[0] = state0
    mass, vol, E, nu, act, seed = (np.ascontiguousarray(np.asarray(a), ft) for a in (mass, vol, E, nu, act, seed))
    aid = np.ascontiguousarray(np.asarray(act_id, np.int32))
    if fp32:
        cc = _Cfg32(cfg.dim, cfg.res, n, cfg.n_act, cfg.dt, (C.c_float * 3)(*cfg.gravity), cfg.bound,
                    (C.c_float * 6)(*cfg.friction), cfg.act_strength, cfg.eps, cfg.material)
    else:
        cc = cfg.c(n)
    err = np.zeros(2, np.int32)
    g0 = np.zeros((n, S), ft)
    gE = np.zeros(n, ft)
    gnu = np.zeros(n, ft)
    ga = np.zeros((max(n_steps, 1), max(cfg.n_act, 1), cfg.dim), ft)
    fwd = L.orc_forward_omp if omp else L.orc_forward
    bwd = L.orc_backward_omp if omp else L.orc_backward
    t0 = time.perf_counter()
    rc = fwd(C.byref(cc), n_steps, cp(traj), cp(mass), cp(vol), cp(E), cp(nu), _i(aid), cp(act), _i(err))
    t1 = time.perf_counter()
    if rc:
        raise OracleError(rc, tuple(err))
    rc = bwd(C.byref(cc), n_steps, cp(traj), cp(mass), cp(vol), cp(E), cp(nu), _i(aid), cp(act), cp(seed),
             cp(g0), cp(gE), cp(gnu), cp(ga))
    t2 = time.perf_counter()
    if rc:
        raise OracleError(rc)
    return t1 - t0, t2 - t0, g0
