"""Thin ctypes binding of the C ABI in ``include/mpm.h`` (library ``libmpm.so``, sm_100a).

Argument marshalling only: every step of the differentiable MLS-MPM path runs in the CUDA
kernels of ``csrc/``.  There is no CPU fallback: ``load()`` raises if the library is
missing, and every call raises ``MPMError`` on a non-zero status.

Arrays may be numpy arrays (host) or torch tensors (host or CUDA); they are passed to the
library as raw pointers (the library detects host vs device memory).  Outputs default to
new numpy arrays; pass ``out=`` tensors to keep results on the device.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpm.so")

STATUS = {0: "MPM_OK", 1: "MPM_ERR_INVALID_ARG", 2: "MPM_ERR_OOM", 3: "MPM_ERR_CUDA",
          4: "MPM_ERR_OUT_OF_DOMAIN", 5: "MPM_ERR_INVERTED", 6: "MPM_ERR_TAPE_FULL",
          7: "MPM_ERR_CALL_ORDER", 8: "MPM_ERR_COMM", 9: "MPM_ERR_OUT_OF_SLAB",
          10: "MPM_ERR_CFL", 11: "MPM_ERR_MIGRATE"}

# every symbol include/mpm.h declares
EXPORTS = ("mpm_create", "mpm_destroy", "mpm_set_state", "mpm_set_actuation", "mpm_forward",
           "mpm_tape_length", "mpm_rewind", "mpm_get_state", "mpm_backward", "mpm_grad",
           "mpm_last_error", "mpm_get_binning", "mpm_get_grid", "mpm_set_profiling",
           "mpm_get_profile", "mpm_launch_count", "mpm_get_step_info", "mpm_grad_mass",
           "mpm_add_seed", "mpm_clear_seeds", "mpm_enable_mass_grad", "mpm_set_slab",
           "mpm_comm_unique_id", "mpm_comm_init", "mpm_group_forward", "mpm_group_backward",
           "mpm_set_controller", "mpm_grad_controller", "mpm_set_graphs", "mpm_set_slab_migrating",
           "mpm_set_transport")


# int fn(void* user, int32 kind, const float* send_l, const float* send_r, float* recv_l,
#        float* recv_r, size_t bytes)   (include/mpm.h mpm_transport_fn)
_TRANSPORT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_size_t)


class MPMError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.status = STATUS.get(code, str(code))
        super().__init__(f"{self.status}: {msg}")


class _Config(C.Structure):
    _fields_ = [("dim", C.c_int32), ("res", C.c_int32), ("batch", C.c_int32),
                ("n_particles", C.c_int32), ("max_steps", C.c_int32), ("n_actuators", C.c_int32),
                ("dt", C.c_float), ("gravity", C.c_float * 3), ("bound", C.c_int32),
                ("friction", C.c_float * 6), ("act_strength", C.c_float), ("device", C.c_int32),
                ("stream", C.c_void_p), ("grid_slots", C.c_int32), ("checkpoint_every", C.c_int32),
                ("material", C.c_int32), ("fuse_g2p2g", C.c_int32)]


_lib = None


def _bundled_nccl():
    """Path of the libnccl.so.2 of the nvidia-nccl wheel torch links against, or None (found
    without importing torch).  libmpm dlopens NCCL lazily; loading this one keeps a later
    `import torch` from resolving its libnccl.so.2 to an older system copy."""
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    return None


def load():
    """Load libmpm.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    if "MPM_NCCL_LIB" not in os.environ:  # the NCCL torch bundles (see nccl_api in mpm_api.cu)
        nccl = _bundled_nccl()
        if nccl:
            os.environ["MPM_NCCL_LIB"] = nccl
    L = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.mpm_create.argtypes = [C.POINTER(_Config), C.POINTER(vp)]
    L.mpm_destroy.argtypes = [vp]
    L.mpm_destroy.restype = None
    L.mpm_set_state.argtypes = [vp] * 10
    L.mpm_set_actuation.argtypes = [vp, vp]
    L.mpm_forward.argtypes = [vp, i32]
    L.mpm_tape_length.argtypes = [vp]
    L.mpm_tape_length.restype = i32
    L.mpm_rewind.argtypes = [vp, i32]
    L.mpm_get_state.argtypes = [vp, i32, vp, vp, vp, vp]
    L.mpm_backward.argtypes = [vp, vp, vp, vp, vp]
    L.mpm_grad.argtypes = [vp] * 8
    L.mpm_last_error.argtypes = [vp]
    L.mpm_last_error.restype = C.c_char_p
    L.mpm_get_binning.argtypes = [vp, i32, vp, vp, vp, vp, vp]
    L.mpm_get_grid.argtypes = [vp, i32, vp, vp]
    L.mpm_set_profiling.argtypes = [vp, i32]
    L.mpm_set_graphs.argtypes = [vp, i32]
    L.mpm_get_profile.argtypes = [vp, C.POINTER(i32), vp, vp, C.c_char_p, i32]
    L.mpm_get_step_info.argtypes = [vp, i32, vp]
    L.mpm_grad_mass.argtypes = [vp, vp]
    L.mpm_enable_mass_grad.argtypes = [vp, i32]
    L.mpm_add_seed.argtypes = [vp, i32, vp, vp, vp, vp]
    L.mpm_clear_seeds.argtypes = [vp]
    L.mpm_launch_count.argtypes = [vp]
    L.mpm_launch_count.restype = i64
    L.mpm_set_controller.argtypes = [vp, vp, vp, vp]
    L.mpm_grad_controller.argtypes = [vp, vp, vp, vp]
    L.mpm_set_slab.argtypes = [vp, i32, i32, i32]
    L.mpm_set_slab_migrating.argtypes = [vp, i32, i32, i32, i32, i32]
    L.mpm_set_transport.argtypes = [vp, _TRANSPORT_FN, vp]
    L.mpm_comm_unique_id.argtypes = [C.c_char_p]
    L.mpm_comm_init.argtypes = [vp, i32, i32, C.c_char_p]
    L.mpm_group_forward.argtypes = [C.POINTER(vp), i32, i32]
    L.mpm_group_backward.argtypes = [C.POINTER(vp), i32] + [C.POINTER(vp)] * 4
    for name in EXPORTS:
        getattr(L, name)
    _lib = L
    return L


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def _check_tensor(a, dtype, n, device, name):
    """A torch tensor passed as a raw pointer: its element type, size, layout and device must
    be what the ABI reads or writes (the library cannot see any of them)."""
    import torch
    want = {np.float32: torch.float32, np.int32: torch.int32}[dtype]
    if a.dtype != want:
        raise TypeError(f"{name}: dtype {a.dtype}, the ABI needs {want}")
    if a.numel() != n:
        raise ValueError(f"{name}: {a.numel()} elements, the ABI needs {n}")
    if not a.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if a.device.type == "cuda" and device is not None and a.device.index != device:
        raise ValueError(f"{name}: on cuda:{a.device.index}, the context is on cuda:{device}")
    if a.device.type not in ("cpu", "cuda"):
        raise ValueError(f"{name}: unsupported device {a.device}")


def _in(a, dtype, shape, device=None, name="input"):
    """An input array: numpy (converted to dtype, made contiguous) or a torch tensor (checked)."""
    if a is None:
        return None
    n = int(np.prod(shape))
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a, dtype=dtype)
        if a.size != n:
            raise ValueError(f"{name}: shape {a.shape}, the ABI needs {n} elements {tuple(shape)}")
        return a
    if hasattr(a, "data_ptr"):
        _check_tensor(a, dtype, n, device, name)
        return a
    raise TypeError(f"{name}: unsupported array type {type(a)}")


def _out(a, dtype, shape, device=None, name="output"):
    """An output buffer the library writes into: numpy (exact dtype, C-contiguous, writeable)
    or a torch tensor (checked)."""
    if a is None:
        return None
    n = int(np.prod(shape))
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags.c_contiguous or not a.flags.writeable or a.size != n:
            raise ValueError(f"{name}: needs a writeable C-contiguous {np.dtype(dtype)} array of {n} elements, "
                             f"got {a.dtype} {a.shape}")
        return a
    if hasattr(a, "data_ptr"):
        _check_tensor(a, dtype, n, device, name)
        return a
    raise TypeError(f"{name}: unsupported array type {type(a)}")


@dataclass
class Config:
    dim: int
    res: int
    batch: int
    n_particles: int
    max_steps: int
    dt: float
    n_actuators: int = 0
    gravity: tuple = (0.0, 0.0, 0.0)
    bound: int = 3
    friction: tuple = (0.0,) * 6
    act_strength: float = 0.0
    device: int = 0
    stream: int = 0
    grid_slots: int = 0
    checkpoint_every: int = 0  # NEXT N2: 0 = full memo; k = k-step segments + checkpoints
    material: int = 0          # NEXT N3: 0 = neo-Hookean (R1), 1 = fixed-corotated (R21)
    fuse_g2p2g: int = 0        # NEXT N2: 1 = fused forward (one particle pass per step)

    @classmethod
    def from_scene(cls, sc, max_steps=None, **kw):
        return cls(dim=sc.dim, res=sc.res, batch=sc.batch, n_particles=sc.n,
                   max_steps=max_steps or sc.steps, dt=sc.dt, n_actuators=sc.n_act,
                   gravity=tuple(sc.gravity), bound=sc.bound, friction=tuple(sc.friction),
                   act_strength=sc.act_strength, **kw)

    def c(self) -> _Config:
        g = list(self.gravity) + [0.0] * (3 - len(self.gravity))
        f = list(self.friction) + [0.0] * (6 - len(self.friction))
        return _Config(self.dim, self.res, self.batch, self.n_particles, self.max_steps,
                       self.n_actuators, self.dt, (C.c_float * 3)(*g[:3]), self.bound,
                       (C.c_float * 6)(*f[:6]), self.act_strength, self.device,
                       self.stream or None, self.grid_slots, self.checkpoint_every, self.material,
                       self.fuse_g2p2g)


class MPM:
    """One simulation context (one GPU, B rollouts).  Mirrors the C ABI one to one."""

    def __init__(self, cfg: Config):
        self.L = load()
        self.cfg = cfg
        self._cc = cfg.c()
        h = C.c_void_p()
        self._check(self.L.mpm_create(C.byref(self._cc), C.byref(h)), h)
        self.h = h

    # -- plumbing -----------------------------------------------------------------------
    def _check(self, rc, h=None):
        if rc != 0:
            hh = h if h is not None else self.h
            msg = self.L.mpm_last_error(hh if hh and hh.value else None).decode()
            raise MPMError(rc, msg)

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.L.mpm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def NT(self):
        """Storage capacity (batch x n_particles)."""
        return self.cfg.batch * self.cfg.n_particles

    @property
    def NU(self):
        """Length of the user-order arrays: NT, or the whole body's count in migrating slab mode."""
        return getattr(self, "_nu", None) or self.NT

    # -- the path -----------------------------------------------------------------------
    def set_state(self, x, v=None, F=None, C_=None, mass=None, vol=None, E=None, nu=None,
                  actuator_id=None):
        d, NT, dev = self.cfg.dim, self.NU, self.cfg.device
        arrs = [_in(x, np.float32, (NT, d), dev, "x"), _in(v, np.float32, (NT, d), dev, "v"),
                _in(F, np.float32, (NT, d, d), dev, "F"), _in(C_, np.float32, (NT, d, d), dev, "C"),
                _in(mass, np.float32, (NT,), dev, "mass"), _in(vol, np.float32, (NT,), dev, "vol"),
                _in(E, np.float32, (NT,), dev, "E"), _in(nu, np.float32, (NT,), dev, "nu"),
                _in(actuator_id, np.int32, (NT,), dev, "actuator_id")]
        self._check(self.L.mpm_set_state(self.h, *[_ptr(a) for a in arrs]))

    def set_scene(self, sc):
        self.set_state(sc.x, sc.v, sc.F, sc.C, sc.mass, sc.vol, sc.E, sc.nu, sc.actuator_id)
        if sc.n_act > 0:
            a = np.zeros((sc.batch, self.cfg.max_steps, sc.n_act, sc.dim), np.float32)
            T = min(self.cfg.max_steps, sc.act.shape[1])
            a[:, :T] = sc.act[:, :T]
            self.set_actuation(a)

    def set_actuation(self, a):
        cfg = self.cfg
        a = _in(a, np.float32, (cfg.batch, cfg.max_steps, cfg.n_actuators, cfg.dim), cfg.device, "actuation")
        self._check(self.L.mpm_set_actuation(self.h, _ptr(a)))

    def forward(self, n_steps: int):
        self._check(self.L.mpm_forward(self.h, int(n_steps)))

    def rewind(self, t: int = 0):
        self._check(self.L.mpm_rewind(self.h, int(t)))

    @property
    def tape_length(self) -> int:
        return self.L.mpm_tape_length(self.h)

    def get_state(self, t: int, out=None):
        d, NT = self.cfg.dim, self.NU
        if out is None:
            out = (np.empty((NT, d), np.float32), np.empty((NT, d), np.float32),
                   np.empty((NT, d, d), np.float32), np.empty((NT, d, d), np.float32))
        shapes = ((NT, d), (NT, d), (NT, d, d), (NT, d, d))
        out = tuple(_out(a, np.float32, sh, self.cfg.device, nm) for a, sh, nm in zip(out, shapes, "xvFC"))
        self._check(self.L.mpm_get_state(self.h, int(t), *[_ptr(a) for a in out]))
        return out

    def backward(self, dLdx=None, dLdv=None, dLdF=None, dLdC=None):
        d, NT, dev = self.cfg.dim, self.NU, self.cfg.device
        arrs = [_in(dLdx, np.float32, (NT, d), dev, "dLdx"), _in(dLdv, np.float32, (NT, d), dev, "dLdv"),
                _in(dLdF, np.float32, (NT, d, d), dev, "dLdF"), _in(dLdC, np.float32, (NT, d, d), dev, "dLdC")]
        self._check(self.L.mpm_backward(self.h, *[_ptr(a) for a in arrs]))

    def grad(self, out=None):
        cfg = self.cfg
        d, NT = cfg.dim, self.NU
        if out is None:
            out = dict(dx0=np.empty((NT, d), np.float32), dv0=np.empty((NT, d), np.float32),
                       dF0=np.empty((NT, d, d), np.float32), dC0=np.empty((NT, d, d), np.float32),
                       dE=np.empty(NT, np.float32), dnu=np.empty(NT, np.float32),
                       da=np.empty((cfg.batch, cfg.max_steps, max(cfg.n_actuators, 0), d), np.float32))
        keys = ("dx0", "dv0", "dF0", "dC0", "dE", "dnu", "da")
        shapes = dict(dx0=(NT, d), dv0=(NT, d), dF0=(NT, d, d), dC0=(NT, d, d), dE=(NT,), dnu=(NT,),
                      da=(cfg.batch, cfg.max_steps, max(cfg.n_actuators, 0), d))
        unknown = set(out) - set(keys)
        if unknown:
            raise KeyError(f"grad(out=): unknown keys {sorted(unknown)}")
        ptrs = [_ptr(_out(out.get(k), np.float32, shapes[k], cfg.device, k)) for k in keys]
        self._check(self.L.mpm_grad(self.h, *ptrs))
        return out

    def enable_mass_grad(self, on: bool = True):
        self._check(self.L.mpm_enable_mass_grad(self.h, 1 if on else 0))

    def grad_mass(self, out=None):
        """dL/dm_p (NEXT N3) from the last backward, user order [B*N]."""
        if out is None:
            out = np.empty(self.NU, np.float32)
        out = _out(out, np.float32, (self.NU,), self.cfg.device, "dmass")
        self._check(self.L.mpm_grad_mass(self.h, _ptr(out)))
        return out

    def add_seed(self, t, dLdx=None, dLdv=None, dLdF=None, dLdC=None):
        """Additive seed dL/dstate_t for a running loss (NEXT N4)."""
        d, NT, dev = self.cfg.dim, self.NU, self.cfg.device
        arrs = [_in(dLdx, np.float32, (NT, d), dev, "dLdx"), _in(dLdv, np.float32, (NT, d), dev, "dLdv"),
                _in(dLdF, np.float32, (NT, d, d), dev, "dLdF"), _in(dLdC, np.float32, (NT, d, d), dev, "dLdC")]
        self._check(self.L.mpm_add_seed(self.h, int(t), *[_ptr(a) for a in arrs]))

    def clear_seeds(self):
        self._check(self.L.mpm_clear_seeds(self.h))

    # -- NEXT N1: closed-loop controller a_t = tanh(W z_t + b) ----------------------------
    @property
    def n_obs(self) -> int:
        return self.cfg.dim * (1 + 2 * self.cfg.n_actuators)

    def set_controller(self, W, b=None, target=None):
        """W [K*d][nz], b [K*d], target [d] (nz = d (1 + 2K)); W=None switches it off."""
        if W is None:
            self._check(self.L.mpm_set_controller(self.h, None, None, None))
            return
        KD = self.cfg.n_actuators * self.cfg.dim
        dev = self.cfg.device
        arrs = [_in(W, np.float32, (KD, self.n_obs), dev, "W"), _in(b, np.float32, (KD,), dev, "b"),
                _in(target, np.float32, (self.cfg.dim,), dev, "target")]
        self._check(self.L.mpm_set_controller(self.h, *[_ptr(a) for a in arrs]))

    def grad_controller(self):
        """(dL/dW, dL/db, dL/dtarget) from the last backward with the controller on."""
        KD = self.cfg.n_actuators * self.cfg.dim
        out = (np.empty((KD, self.n_obs), np.float32), np.empty(KD, np.float32),
               np.empty(self.cfg.dim, np.float32))
        self._check(self.L.mpm_grad_controller(self.h, *[_ptr(a) for a in out]))
        return out

    # -- slab mode -----------------------------------------------------------
    def set_slab_migrating(self, x_lo: int, x_hi: int, halo_blocks: int, n_global: int, mig_cap: int = 0):
        """Migrating slab mode (include/mpm.h): ownership by base_x at every step, particles
        migrate between neighbouring slabs; user arrays span the whole body (n_global)."""
        self._check(self.L.mpm_set_slab_migrating(self.h, int(x_lo), int(x_hi), int(halo_blocks), int(n_global),
                                                  int(mig_cap)))
        self._nu = int(n_global)

    def set_transport(self, fn):
        """Host-staged slab exchanges through fn(kind, send_l, send_r, recv_l, recv_r) with numpy
        float32 views (None on a side without a neighbour); kind "reduce": overwrite send_l with
        the sum over ranks.  fn=None unsets."""
        if fn is None:
            self._transport = None
            self._check(self.L.mpm_set_transport(self.h, None, None))
            return
        kinds = {0: "window", 1: "migrate", 2: "migrate_adj", 3: "reduce"}

        def cb(user, kind, sl, sr, rl, rr, nbytes):
            try:
                n = nbytes // 4
                view = lambda p: None if not p else np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), (n,))
                fn(kinds[kind], view(sl), view(sr), view(rl), view(rr))
                return 0
            except Exception as e:  # noqa: BLE001 -- reported through the status code
                import traceback
                traceback.print_exc()
                return 1
        self._transport = _TRANSPORT_FN(cb)  # keep alive while set
        self._check(self.L.mpm_set_transport(self.h, self._transport, None))

    def set_slab(self, x_lo: int, x_hi: int, halo_blocks: int = 1):
        """This context simulates the x-slab [x_lo, x_hi) of node planes (before set_state)."""
        self._check(self.L.mpm_set_slab(self.h, int(x_lo), int(x_hi), int(halo_blocks)))

    def comm_init(self, rank: int, world: int, uid: bytes):
        """Join the NCCL halo-exchange communicator (ranks ordered by slab; collective)."""
        assert len(uid) == 128
        self._check(self.L.mpm_comm_init(self.h, int(rank), int(world), uid))

    # -- introspection -------------------------------------------------------------------
    def get_binning(self, t: int):
        cfg = self.cfg
        d, NT = cfg.dim, self.NT
        Bb = 4 if d == 3 else 8
        nb = (cfg.res // Bb) ** d
        x = np.empty((NT, d), np.float32)
        orig = np.empty(NT, np.int32)
        key = np.empty(NT, np.int32)
        perm = np.empty(NT, np.int32)
        bs = np.empty(cfg.batch * nb + 1, np.int32)
        self._check(self.L.mpm_get_binning(self.h, int(t), _ptr(x), _ptr(orig), _ptr(key),
                                           _ptr(perm), _ptr(bs)))
        return x, orig, key, perm, bs

    def get_grid(self, t: int):
        cfg = self.cfg
        nn = cfg.res ** cfg.dim
        m = np.empty((cfg.batch, nn), np.float32)
        vbar = np.empty((cfg.batch, nn, cfg.dim), np.float32)
        self._check(self.L.mpm_get_grid(self.h, int(t), _ptr(m), _ptr(vbar)))
        return m, vbar

    def step_info(self, t: int):
        """(occupied blocks, touched blocks, first arena slot) of tape step t."""
        out = np.zeros(3, np.int32)
        self._check(self.L.mpm_get_step_info(self.h, int(t), _ptr(out)))
        return tuple(int(v) for v in out)

    def set_profiling(self, on: bool):
        self._check(self.L.mpm_set_profiling(self.h, 1 if on else 0))

    def launch_count(self) -> int:
        """Kernels launched by this context so far (include/mpm.h mpm_launch_count)."""
        return int(self.L.mpm_launch_count(self.h))

    def set_graphs(self, on: bool = True):
        """Replay the step loops as CUDA graphs (include/mpm.h mpm_set_graphs; needs
        Config.stream)."""
        self._check(self.L.mpm_set_graphs(self.h, 1 if on else 0))

    def profile(self):
        n = C.c_int32(32)
        ms = np.zeros(32, np.float32)
        cnt = np.zeros(32, np.int64)
        names = C.create_string_buffer(1024)
        self._check(self.L.mpm_get_profile(self.h, C.byref(n), _ptr(ms), _ptr(cnt), names, 1024))
        keys = names.value.decode().split(";")
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(keys[:n.value])}

    @property
    def launches(self) -> int:
        return int(self.L.mpm_launch_count(self.h))


def comm_unique_id() -> bytes:
    """128-byte NCCL unique id for mpm_comm_init (create on one rank, broadcast to all)."""
    L = load()
    buf = C.create_string_buffer(128)
    rc = L.mpm_comm_unique_id(buf)
    if rc != 0:
        raise MPMError(rc, "ncclGetUniqueId failed")
    return buf.raw


def _group_check(sims, rc):
    if rc != 0:
        msgs = [s.L.mpm_last_error(s.h).decode() for s in sims]
        raise MPMError(rc, " | ".join(m for m in msgs if m) or "group call failed")


def _handles(sims):
    return (C.c_void_p * len(sims))(*[s.h.value for s in sims])


def group_forward(sims, n_steps: int):
    """Advance adjacent slab contexts of one process in lockstep (single-GPU slab emulation)."""
    L = load()
    _group_check(sims, L.mpm_group_forward(_handles(sims), len(sims), int(n_steps)))


def group_backward(sims, dLdx=None, dLdv=None, dLdF=None, dLdC=None):
    """Reverse mode over adjacent slab contexts; seeds are lists (one array per context)."""
    L = load()
    keep = []

    def arr(seeds, shape_of):
        if seeds is None:
            return None
        ptrs = []
        for s, a in zip(sims, seeds):
            a = _in(a, np.float32, shape_of(s), s.cfg.device, "seed")
            keep.append(a)
            ptrs.append(_ptr(a))
        return (C.c_void_p * len(sims))(*ptrs)

    vec = lambda s: (s.NU, s.cfg.dim)
    mat = lambda s: (s.NU, s.cfg.dim, s.cfg.dim)
    args = [arr(dLdx, vec), arr(dLdv, vec), arr(dLdF, mat), arr(dLdC, mat)]
    _group_check(sims, L.mpm_group_backward(_handles(sims), len(sims), *args))
