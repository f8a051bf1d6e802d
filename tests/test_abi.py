"""The C-ABI library builds, loads and exports every symbol include/mpm.h declares; config
validation happens before any CUDA call.  CPU only (no compute calls)."""
import ctypes as C
import os
import re

import pytest

from paper_1810_01054_b200 import build, mpm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mpm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    build.build()
    L = mpm.load()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(mpm.EXPORTS)


@pytest.mark.parametrize("bad", [
    dict(dim=4), dict(res=100), dict(res=8), dict(batch=0), dict(n_particles=0),
    dict(max_steps=0), dict(n_actuators=-1), dict(dt=0.0), dict(bound=40),
    dict(material=2), dict(checkpoint_every=-1), dict(checkpoint_every=5), dict(fuse_g2p2g=2),
])
def test_config_validation_is_host_side(bad):
    kw = dict(dim=3, res=64, batch=1, n_particles=10, max_steps=4, dt=1e-4)
    kw.update(bad)
    cfg = mpm.Config(**kw)
    with pytest.raises(mpm.MPMError) as e:
        mpm.MPM(cfg)
    assert e.value.status == "MPM_ERR_INVALID_ARG"
    # the reason survives the failed create (mpm_last_error(NULL), thread-local)
    msg = str(e.value)
    assert "create failed" not in msg and "null context" not in msg and len(msg) > 30, msg


def test_no_cpu_fallback(monkeypatch, tmp_path):
    """The binding refuses to run without the CUDA library (no silent fallback)."""
    monkeypatch.setattr(mpm, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(mpm, "_lib", None)
    with pytest.raises(ImportError):
        mpm.load()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1810_01054_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "mpm_oracle" not in txt and "liboracle" not in txt, f


def test_binding_checks_dtype_size_layout_and_device():
    """The binding passes raw pointers, so it must reject what the ABI would misread: a torch
    tensor of the wrong dtype (an int64 actuator id read as int32, an fp64 x read as fp32), the
    wrong size, a non-contiguous view, a tensor on another GPU; and output buffers that numpy
    would have to convert (the library would write into a temporary)."""
    import numpy as np
    import torch
    from paper_1810_01054_b200.mpm import _in, _out
    assert _in(np.zeros((3, 2), np.float64), np.float32, (3, 2)).dtype == np.float32  # numpy: converted
    with pytest.raises(TypeError):
        _in(torch.zeros(6, dtype=torch.float64), np.float32, (3, 2))
    with pytest.raises(TypeError):
        _in(torch.zeros(3, dtype=torch.int64), np.int32, (3,))
    with pytest.raises(ValueError):
        _in(torch.zeros(5, dtype=torch.float32), np.float32, (3, 2))
    with pytest.raises(ValueError):
        _in(torch.zeros(6, 2, dtype=torch.float32)[:, 0], np.float32, (6,))
    with pytest.raises(ValueError):
        _in(np.zeros(4, np.float32), np.float32, (3,))
    assert _in(torch.zeros(6, dtype=torch.float32), np.float32, (3, 2)) is not None
    with pytest.raises(ValueError):
        _out(np.zeros((3, 2), np.float64), np.float32, (3, 2))
    with pytest.raises(ValueError):
        _out(np.zeros((2, 3), np.float32).T, np.float32, (3, 2))
    with pytest.raises(TypeError):
        _out(torch.zeros(6, dtype=torch.float64), np.float32, (3, 2))
    assert _out(np.zeros((3, 2), np.float32), np.float32, (3, 2)) is not None
    with pytest.raises(TypeError):
        _in([1.0, 2.0], np.float32, (2,))


def test_bundled_nccl_lookup():
    """The binding points libmpm's lazy NCCL load at the nvidia-nccl wheel torch bundles (so a
    later `import torch` keeps its libnccl.so.2), found without importing torch."""
    from paper_1810_01054_b200 import mpm
    p = mpm._bundled_nccl()
    assert p is None or (os.path.basename(p) == "libnccl.so.2" and os.path.exists(p))
